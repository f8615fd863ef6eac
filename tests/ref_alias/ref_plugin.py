"""pytest plugin for the vendored reference suite: the documented deviations.

Every reference test runs unchanged against paper_1407_6603_b200 (through
the `wordsort` alias). The tests listed here assert properties of the
reference's CPU thread pool (wall-clock speedups from more worker threads),
which a GPU sort that ignores `threads` cannot show; they are marked xfail
with the reason, not skipped, so their outcome stays visible."""
import pytest

DEVIATIONS = {
    # node-id suffix -> reason
    "test_acceptance.py::test_criterion_8_scaling_smoke":
        "grows the corpus until a 1-thread sort takes >= 5 s, then expects more threads to be "
        "faster: the GPU sorts 3M words in milliseconds and ignores `threads`",
    "test_parallel.py::test_worker_count_capped_by_bucket_count":
        "counts threading.Thread workers: sort_all_parallel is one segmented device launch "
        "over all buckets (engine.py:140-201's pool replaced), it spawns no threads",
}


def pytest_collection_modifyitems(config, items):
    for item in items:
        for key, reason in DEVIATIONS.items():
            if item.nodeid.endswith(key):
                item.add_marker(pytest.mark.xfail(reason=reason, strict=False))
