"""compute-sanitizer over a small end-to-end case of the hot path (race detection /
sanitizers): memcheck (out-of-bounds and misaligned global/shared accesses, leaks of device
allocations are not checked — the stream-ordered pool keeps blocks), racecheck (shared-memory
hazards) and synccheck (illegal barrier use).  The case (tools/sanitize_case.py) runs
quantize, the kernel map (sorted rows, cooperative sort, PDL launches), bf16 + fp32 conv
forward/backward, a strided map with pooling and a transposed conv."""
import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    san = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(san):
        pytest.skip("compute-sanitizer not installed")
    cmd = [san, "--tool", tool, "--error-exitcode", "99", sys.executable, str(ROOT / "tools" / "sanitize_case.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    if r.returncode != 0 and "compute-sanitizer is closed" in out:
        # the GPU pool's wrapper refuses the tool (it left GPUs needing a reset elsewhere):
        # nothing ran, so there is nothing to judge (round-2 runs before the closure were clean)
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert r.returncode == 0, out[-4000:]
    assert "ok" in r.stdout
    clean = "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out
    assert clean, out[-4000:]
