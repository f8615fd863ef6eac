import json
import sys
from pathlib import Path

import pytest

import os

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
# The library counts distinct words (csrc/dedupe.cu) only for texts of 48 MiB
# and more by default; the suite lowers that to 1 MiB (read once per process,
# before the first library call) so that its mid-size fixtures -- and every
# knob subprocess, which inherits the environment -- go through the counting
# path as well. Tests of the sort paths themselves set WSORT_NO_DEDUPE=1.
os.environ.setdefault("WSORT_DEDUPE_MIN", str(1 << 20))
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_tokenize():
    return json.loads((GOLDEN / "tokenize_kat.json").read_text())


@pytest.fixture(scope="session")
def golden_stats():
    return json.loads((GOLDEN / "stats_kat.json").read_text())


@pytest.fixture(scope="session")
def golden_configs():
    return json.loads((GOLDEN / "configs.json").read_text())


def config_text(rec: dict) -> bytes:
    from paper_1407_6603_b200 import synth

    text = synth.generate(rec["config"])
    if rec.get("prefix_words"):
        text = synth.prefix(text, rec["prefix_words"])
    return text


@pytest.fixture(autouse=True)
def _bounds_checks(request):
    """With WSORT_CHECKED=1 (a library built by tools/checked_build.sh), every
    GPU test also asserts that no kernel bounds check failed during it."""
    yield
    import os

    if os.environ.get("WSORT_CHECKED") != "1" or request.node.get_closest_marker("gpu") is None:
        return
    from paper_1407_6603_b200 import _native

    assert _native.checked_build(), "WSORT_CHECKED=1 but the library is not a checked build"
    fails, where = _native.debug_checks()
    assert fails == 0, f"{fails} device bounds checks failed, first at {where}"


def pytest_unconfigure(config):
    """Last hook of a run (the summary is out). When the CUDA library was
    loaded, leave without interpreter teardown: with the library's worker
    threads and handles alive, teardown has crashed (SIGSEGV after the summary)
    once in a while on the GPU boxes, which would turn a green run red."""
    mod = sys.modules.get("paper_1407_6603_b200._native")
    if mod is None or getattr(mod, "_lib", None) is None:
        return
    status = getattr(config, "_ws_exitstatus", None)
    if status is None:
        return
    sys.stdout.flush()
    sys.stderr.flush()
    os._exit(int(status))


def pytest_sessionfinish(session, exitstatus):
    session.config._ws_exitstatus = exitstatus
