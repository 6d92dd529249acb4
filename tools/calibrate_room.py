"""Calibrate synthetic.ROOM_AREA so that 2 cm quantization gives ~150k voxels on average.

Calls only oracle/ (the CPU oracle) and synthetic/ (the generators); the resulting
constants are hard-coded in synthetic/__init__.py.  Run: python tools/calibrate_room.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import synthetic  # noqa: E402

TARGET = 150_000
for noisy in (False, True):
    a0 = synthetic.ROOM_AREA[noisy]
    n = [oracle.quantize(synthetic.room_points(2000 + s, noisy, area=a0), synthetic.ROOM_VOXEL)[0].shape[0]
         for s in range(8)]
    print(f"noisy={noisy} area={a0} N={n} mean={np.mean(n):.0f} rel.sd={np.std(n) / np.mean(n):.3f} "
          f"suggested area={a0 * TARGET / np.mean(n):.1f}")
