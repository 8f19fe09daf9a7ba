"""The drop-in boundary, proven from the reference side: the reference's own
engine tests (tests/test_engine.cpp:70-109, 139-213, restated without doctest
in integration/test_engine_b200.cpp) built from the UNMODIFIED reference
headers and sources with every float kernel of build_pipeline / run_loss_step
/ pairwise_optimize bound to libmdg by integration/mdreg_b200.hpp.

CPU: the binary was built by integration/Makefile and links libmdg.so.  GPU:
it runs, every case passes, and libmdg launched kernels."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "test_engine_b200")


def _have_bin():
    if not os.path.exists(BIN):
        pytest.skip("integration binary not built (needs the reference tree at build time)")


def test_binary_links_libmdg():
    _have_bin()
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libmdg.so" in out and "not found" not in out.split("libmdg.so")[1].split("\n")[0]


@pytest.mark.gpu
def test_reference_engine_tests_run_on_libmdg(cuda):
    _have_bin()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=1200)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    res = json.loads(line)
    print(json.dumps(res["cases"]), "launches", res["mdg_launches"], "epe",
          res.get("translation_epe"))
    assert res["mdg_launches"] > 1000, res["mdg_launches"]
    failed = [k for k, ok in res["cases"].items() if not ok]
    assert not failed, (failed, r.stderr[-2000:])
    assert r.returncode == 0
