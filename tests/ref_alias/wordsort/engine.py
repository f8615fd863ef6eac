import sys

from paper_1407_6603_b200 import engine as _m

if __name__ == "__main__":  # python -m wordsort.engine
    sys.exit(_m.main())
sys.modules[__name__] = _m
