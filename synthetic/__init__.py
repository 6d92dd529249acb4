"""Seeded synthetic workloads shared by the tests, bench.py and smoke().

This module holds NONE of the method's arithmetic: it only draws random points,
integer cells, features and weights.  Quantization, hashing, kernel maps and
convolutions live in the CUDA path (``paper_1904_08755_b200``) and, independently, in
the oracle (``oracle/``).  Recipes follow SURVEY.md §8(d) and DESIGN.md §4; every
generator is deterministic given its seed (numpy PCG64).

Workload shapes (BASELINE.json configs):
  cfg1  2,000 distinct cells of a 32^3 grid (integer coordinates).
  cfg2  ScanNet-like indoor room sampled as float points, quantized at 2 cm to ~150k voxels.
  cfg3  Synthia-like outdoor 3-frame video, ~100k voxels per frame at 0.2 m.
  cfg4  cfg2's coordinates (stride-2 encoder / decoder layer pair).
  cfg5  16 rooms (batch indices 0..15).
"""
from __future__ import annotations

import numpy as np

ROOM_VOXEL = 0.02     # 2 cm (Table 1 "2cm")
VIDEO_VOXEL = 0.2     # outdoor video voxel


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


# ----------------------------------------------------------------------------- cfg1
def random_cells(seed: int, n: int = 2000, grid: int = 32, D: int = 3, batch: int = 0) -> np.ndarray:
    """n distinct cells sampled without replacement from grid^D; int32 [n][D+1], batch last."""
    g = rng(seed)
    flat = g.choice(grid ** D, size=n, replace=False)
    cells = np.stack(np.unravel_index(flat, (grid,) * D), axis=1).astype(np.int32)
    return np.concatenate([cells, np.full((n, 1), batch, np.int32)], axis=1)


# ----------------------------------------------------------------------------- surfaces
def _plane(g, origin, u, v, density, holes=()):
    """Uniform points on the parallelogram origin + s*u + t*v, s,t in [0,1)."""
    u = np.asarray(u, np.float64)
    v = np.asarray(v, np.float64)
    area = float(np.linalg.norm(np.cross(u, v)))
    n = int(g.poisson(area * density))
    st = g.random((n, 2))
    keep = np.ones(n, bool)
    for (s0, s1, t0, t1) in holes:
        keep &= ~((st[:, 0] >= s0) & (st[:, 0] < s1) & (st[:, 1] >= t0) & (st[:, 1] < t1))
    st = st[keep]
    return np.asarray(origin, np.float64) + st[:, :1] * u + st[:, 1:] * v


def _box(g, center, size, yaw, density, bottom=False):
    cx, cy, cz = center
    sx, sy, sz = size
    c, s = np.cos(yaw), np.sin(yaw)
    ex = np.array([c, s, 0.0]) * sx
    ey = np.array([-s, c, 0.0]) * sy
    ez = np.array([0.0, 0.0, sz])
    o = np.array([cx, cy, cz]) - ex / 2 - ey / 2
    faces = [(o + ez, ex, ey), (o, ex, ez), (o + ey, ex, ez), (o, ey, ez), (o + ex, ey, ez)]
    if bottom:
        faces.append((o, ex, ey))
    return np.concatenate([_plane(g, *f, density) for f in faces])


def _cylinder(g, center, radius, height, density):
    area = 2 * np.pi * radius * height + np.pi * radius ** 2
    n = int(g.poisson(area * density))
    side = g.random(n) < (2 * np.pi * radius * height) / area
    th = g.random(n) * 2 * np.pi
    z = np.where(side, g.random(n) * height, height)
    r = np.where(side, radius, radius * np.sqrt(g.random(n)))
    return np.stack([center[0] + r * np.cos(th), center[1] + r * np.sin(th), center[2] + z], axis=1)


# ----------------------------------------------------------------------------- cfg2
# Total surface area (m^2) of a room; chosen once (tools/calibrate_room.py, which calls
# only oracle/) so that quantization at 2 cm yields N ~ 150k voxels.
ROOM_AREA = {False: 69.7, True: 58.1}
ROOM_DENSITY = 8000.0  # points per m^2 (>= 3 per (2 cm)^2 patch)


def room_points(seed: int, noisy: bool = False, area: float | None = None) -> np.ndarray:
    """ScanNet-like indoor room ("entire room ... without cropping") as float32 [N_p][3].

    Floor + 4 walls (2.4-3 m high, door/window openings) + pieces of furniture
    (5-12 boxes, cylinders, tilted planes), centred on the origin so that negative coordinates
    are exercised.  The footprint is scaled so that the total surface area equals
    ``area`` (default ROOM_AREA[noisy]), which pins the voxel count near 150k at 2 cm.
    ``noisy`` adds N(0, 2 mm) jitter (the noisy ScanNet variant).
    """
    g = rng(seed)
    target = ROOM_AREA[noisy] if area is None else area
    W0, L0, H = g.uniform(4.0, 5.5), g.uniform(5.0, 6.5), g.uniform(2.4, 3.0)
    items = []
    for _ in range(int(g.integers(5, 13))):
        kind = g.random()
        fx, fy = g.random(), g.random()
        if kind < 0.6:
            sx, sy, sz = g.uniform(0.3, 1.2), g.uniform(0.3, 0.9), g.uniform(0.3, 0.9)
            items.append(("box", fx, fy, (sx, sy, sz), g.uniform(0, np.pi)))
        elif kind < 0.85:
            items.append(("cyl", fx, fy, g.uniform(0.15, 0.4), g.uniform(0.4, 1.0)))
        else:
            yaw, tilt = g.uniform(0, np.pi), g.uniform(0.3, 1.2)
            items.append(("tilt", fx, fy, yaw, tilt, g.uniform(0.8, 1.6), g.uniform(0.6, 1.2)))
    doors = (g.uniform(0.1, 0.7), [g.uniform(0.1, 0.6) if g.random() < 0.6 else None for _ in range(4)])
    # Voxel-weighted area: a thin surface with unit normal n crosses ~ area * |n|_1 / v^2
    # voxels, so each furniture surface is weighted by the L1 norm of its normal.
    furn = 0.0
    for it in items:
        if it[0] == "box":
            sx, sy, sz = it[3]
            w1 = abs(np.cos(it[4])) + abs(np.sin(it[4]))
            furn += sx * sy + 2 * (sx + sy) * sz * w1
        elif it[0] == "cyl":
            furn += 2 * np.pi * it[3] * it[4] * (4 / np.pi) + np.pi * it[3] ** 2
        else:
            yaw, tilt = it[3], it[4]
            nrm = np.cross([np.cos(yaw), np.sin(yaw), 0.0],
                           [-np.sin(yaw) * np.cos(tilt), np.cos(yaw) * np.cos(tilt), np.sin(tilt)])
            furn += it[5] * it[6] * float(np.abs(nrm).sum() / np.linalg.norm(nrm))
    # weighted area(k) = W0 L0 k^2 + 2 (W0 + L0) H k + furniture (openings are ignored)
    a, b, c = W0 * L0, 2 * (W0 + L0) * H, furn - target
    k = (-b + np.sqrt(b * b - 4 * a * c)) / (2 * a)
    W, L = W0 * k, L0 * k
    dens = ROOM_DENSITY
    x0, y0 = -W / 2, -L / 2
    parts = [_plane(g, (x0, y0, 0.0), (W, 0, 0), (0, L, 0), dens)]
    walls = [((x0, y0, 0), (W, 0, 0)), ((x0, y0 + L, 0), (W, 0, 0)),
             ((x0, y0, 0), (0, L, 0)), ((x0 + W, y0, 0), (0, L, 0))]
    for i, (o, u) in enumerate(walls):
        holes = []
        ln = float(np.linalg.norm(u))
        if i == 0:  # a door
            holes.append((doors[0], doors[0] + 0.9 / ln, 0.0, 2.0 / H))
        if doors[1][i] is not None:  # a window
            holes.append((doors[1][i], doors[1][i] + 1.2 / ln, 0.35, 0.75))
        parts.append(_plane(g, o, u, (0, 0, H), dens, holes))
    for it in items:
        cx = x0 + 0.3 + it[1] * max(W - 0.6, 0.1)
        cy = y0 + 0.3 + it[2] * max(L - 0.6, 0.1)
        if it[0] == "box":
            parts.append(_box(g, (cx, cy, 0.0), it[3], it[4], dens))
        elif it[0] == "cyl":
            parts.append(_cylinder(g, (cx, cy, 0.0), it[3], it[4], dens))
        else:  # tilted plane (e.g. a leaning board / sofa back)
            _, _, _, yaw, tilt, lu, lv = it
            u = np.array([np.cos(yaw), np.sin(yaw), 0.0]) * lu
            v = np.array([-np.sin(yaw) * np.cos(tilt), np.cos(yaw) * np.cos(tilt), np.sin(tilt)]) * lv
            parts.append(_plane(g, (cx, cy, 0.0), u, v, dens))
    pts = np.concatenate(parts)
    if noisy:
        pts = pts + g.normal(0.0, 0.002, pts.shape)
    g.shuffle(pts, axis=0)  # sensor order is not spatial order
    return pts.astype(np.float32)


def rooms_batch(seed: int, n_scans: int = 16, noisy: bool = False):
    """cfg5: n_scans rooms (seeds seed..seed+n-1) concatenated; returns (points, batch int32)."""
    pts, bat = [], []
    for b in range(n_scans):
        p = room_points(seed + b, noisy)
        pts.append(p)
        bat.append(np.full(p.shape[0], b, np.int32))
    return np.concatenate(pts), np.concatenate(bat)


# ----------------------------------------------------------------------------- cfg3
VIDEO_DENSITY = 100.0  # points per m^2 (>= 3 per (0.2 m)^2 patch)
VIDEO_RADIUS = 22.0    # visibility radius


def video_points(seed: int, frames: int = 3):
    """Synthia-like outdoor 3D video (50 m scene per step).

    Returns (points float32 [N_p][3] in world frame, frame int32 [N_p]).  Static
    geometry keeps its world coordinates across frames (camera extrinsics); the
    ego vehicle advances ~1 m per frame and sees a 22 m radius; ~15 cars move.
    """
    g = rng(seed)
    dens = VIDEO_DENSITY
    static = [_plane(g, (-25.0, -25.0, 0.1), (50.0, 0, 0), (0, 50.0, 0), dens)]
    for _ in range(20):  # building facades along both sides of the street
        side = 1.0 if g.random() < 0.5 else -1.0
        x = g.uniform(-25, 20)
        y = side * g.uniform(7.0, 12.0)
        w = g.uniform(6.0, 14.0)
        h = g.uniform(6.0, 14.0)
        static.append(_plane(g, (x, y, 0.0), (w, 0, 0), (0, 0, h), dens))
    static = np.concatenate(static)
    cars = [(g.uniform(-20, 20), g.uniform(-5, 5), g.uniform(0, np.pi), g.uniform(-1.5, 1.5)) for _ in range(15)]
    pts, fr = [], []
    for t in range(frames):
        ego = np.array([-5.0 + 1.0 * t, 0.0, 0.0])
        # independent sensor samples per frame: thin the static points and re-jitter within
        # a voxel-scale neighbourhood (a fresh scan of the same surfaces)
        keep = g.random(static.shape[0]) < 0.85
        s = static[keep] + g.uniform(-0.05, 0.05, (int(keep.sum()), 3))
        dyn = []
        for (cx, cy, yaw, vel) in cars:
            c = (cx + vel * t * np.cos(yaw), cy + vel * t * np.sin(yaw), 0.0)
            dyn.append(_box(g, c, (4.2, 1.8, 1.5), yaw, dens))
        frame_pts = np.concatenate([s] + dyn)
        vis = np.linalg.norm(frame_pts[:, :2] - ego[:2], axis=1) < VIDEO_RADIUS
        frame_pts = frame_pts[vis]
        g.shuffle(frame_pts, axis=0)
        pts.append(frame_pts)
        fr.append(np.full(frame_pts.shape[0], t, np.int32))
    return np.concatenate(pts).astype(np.float32), np.concatenate(fr)


# ----------------------------------------------------------------------------- features
def features(seed: int, n: int, c: int) -> np.ndarray:
    """Features U(-1, 1), fp32 [n][c]."""
    return rng(seed).uniform(-1.0, 1.0, (n, c)).astype(np.float32)


def weights(seed: int, K: int, c_out: int, c_in: int) -> np.ndarray:
    """W_i ~ U(+-1/sqrt(C_in * K)) (S:327 fan-in rule), fp32 [K][C_out][C_in]."""
    a = 1.0 / np.sqrt(c_in * K)
    return rng(seed).uniform(-a, a, (K, c_out, c_in)).astype(np.float32)
