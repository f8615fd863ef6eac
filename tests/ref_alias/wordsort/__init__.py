"""`wordsort` -> paper_1407_6603_b200: lets the reference's own test modules
(vendored by tools/vendor_reference.sh into baseline/_ref/ref_tests, never
committed) run unchanged against this package. Test infrastructure only.
Each submodule below replaces itself in sys.modules with the package's
module of the same role (bench -> harness)."""
from paper_1407_6603_b200 import *  # noqa: F401,F403
from paper_1407_6603_b200 import __all__  # noqa: F401
