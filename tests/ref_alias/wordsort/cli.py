import sys

from paper_1407_6603_b200 import cli as _m

if __name__ == "__main__":  # python -m wordsort.cli
    sys.exit(_m.main())
sys.modules[__name__] = _m
