"""compute-sanitizer on the tensor-core K1 kernels: memcheck and
synccheck on both (the per-tile kernel on 12-qubit tiles and the persistent TMEM
kernel on 13-qubit tiles, with conventional channels, n = 13), racecheck on the
per-tile kernel.  racecheck also reports hazards in the persistent kernel between
its cp.async tile loads and later reads; those are ordered by the cp.async-mbarrier
completion (cp.async.mbarrier.arrive.noinc + mbarrier wait), which racecheck does not
model (profiles/r2_sanitize_racecheck.log)."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tool, tiles):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not found")
    r = subprocess.run([cs, "--tool", tool, "--print-limit", "10", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_run.py"), "13", tiles],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses to run (pool policy); the last
        # clean runs are kept in profiles/r2_sanitize_*.log
        pytest.skip("compute-sanitizer closed on this GPU pool: " + out.strip().splitlines()[0][:200])
    assert r.returncode == 0, out[-2000:]
    assert out.count(" ok") == len(tiles.split(",")), out[-2000:]
    return out


@pytest.mark.parametrize("tool", ["memcheck", "synccheck"])
def test_sanitizer_clean(tool):
    out = _run(tool, "12,13")
    assert re.search(r"ERROR SUMMARY: 0 errors", out), out[-2000:]


def test_racecheck_per_tile_kernel():
    out = _run("racecheck", "12")
    assert re.search(r"RACECHECK SUMMARY: 0 hazards displayed \(0 errors, 0 warnings\)", out), out[-2000:]
