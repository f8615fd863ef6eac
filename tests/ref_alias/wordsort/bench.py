import sys

from paper_1407_6603_b200 import harness as _m

sys.modules[__name__] = _m
