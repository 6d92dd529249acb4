"""Pins for the oracle's coordinate functions (O1-O3) against the paper, SPEC worked
examples, brute force and invariants.  No GPU."""
import numpy as np
import pytest

from conftest import full_grid, golden_lines


def test_quantize_worked_examples(orc):
    # tests/golden/quantize_example.txt: S:77 and reading R6.
    for line in golden_lines("quantize_example.txt"):
        lhs, rhs = line.split("->")
        v, *p = [float(x) for x in lhs.split()]
        want = [int(x) for x in rhs.split()]
        coords, p2r, first = orc.quantize(np.array([p], np.float32), v)
        assert coords.tolist() == [want + [0]]
        assert p2r.tolist() == [0] and first.tolist() == [0]


def _brute_voxels(points, voxel, batch):
    """Independent dedup: Python dict keyed by the tuple of floors, first occurrence wins."""
    q = np.floor(points.astype(np.float32) / np.float32(voxel)).astype(np.int64)
    rows, first, p2r = {}, [], []
    for p in range(points.shape[0]):
        key = tuple(q[p].tolist()) + (int(batch[p]),)
        if key not in rows:
            rows[key] = len(rows)
            first.append(p)
        p2r.append(rows[key])
    coords = np.array(list(rows.keys()), np.int64).reshape(-1, points.shape[1] + 1)
    return coords, np.array(p2r), np.array(first)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_quantize_matches_brute_force(orc, seed):
    # voxel count equals the brute-force set of floors; R8/R9 first-occurrence order.
    g = np.random.default_rng(seed)
    pts = g.uniform(-1.0, 1.0, (3000, 3)).astype(np.float32)
    batch = g.integers(0, 3, 3000).astype(np.int32)
    coords, p2r, first = orc.quantize(pts, 0.1, batch)
    bc, bp, bf = _brute_voxels(pts, 0.1, batch)
    assert np.array_equal(coords, bc)
    assert np.array_equal(p2r, bp)
    assert np.array_equal(first, bf)
    # invariants: first point maps to its row; first_point is increasing (first occurrence)
    assert np.array_equal(p2r[first], np.arange(coords.shape[0]))
    assert np.all(np.diff(first) > 0)


def test_quantize_batch_isolation(orc):
    # Eq. 1: identical spatial coordinates in different batches stay distinct.
    pts = np.array([[0.05, 0.05, 0.05]] * 4, np.float32)
    coords, p2r, _ = orc.quantize(pts, 0.1, np.array([0, 1, 0, 1], np.int32))
    assert coords.tolist() == [[0, 0, 0, 0], [0, 0, 0, 1]]
    assert p2r.tolist() == [0, 1, 0, 1]


def test_quantize_errors_and_empty(orc):
    pts = np.array([[0.0, 0.0], [np.nan, 0.0], [np.inf, 1.0]], np.float32)
    with pytest.raises(orc.OracleError) as e:
        orc.quantize(pts, 0.1)
    assert e.value.status == orc.NONFINITE_INPUT and e.value.row == 1
    with pytest.raises(orc.OracleError) as e:
        orc.quantize(np.array([[0.0], [3e9]], np.float32), 1.0)
    assert e.value.status == orc.COORD_RANGE and e.value.row == 1
    coords, p2r, first = orc.quantize(np.zeros((0, 3), np.float32), 0.1)
    assert coords.shape == (0, 4) and p2r.shape == (0,)


def test_create_identity_and_inverse(orc):
    g = np.random.default_rng(5)
    c = np.unique(g.integers(-50, 50, (500, 3)), axis=0)
    c = g.permutation(c)
    rows = np.concatenate([c, np.zeros((c.shape[0], 1), int)], axis=1).astype(np.int32)
    out, inv = orc.create(rows)
    assert np.array_equal(out, rows)  # already-unique input keeps its order
    assert np.array_equal(inv, np.arange(rows.shape[0]))
    dup = np.concatenate([rows, rows[::-1]])
    out2, inv2 = orc.create(dup)
    assert np.array_equal(out2, rows)
    assert np.array_equal(out2[inv2], dup)


def test_create_stride_check(orc):
    rows = np.array([[0, 2, 0], [2, 3, 0]], np.int32)
    with pytest.raises(orc.OracleError) as e:
        orc.create(rows, tensor_stride=[2, 2])
    assert e.value.status == orc.STRIDE and e.value.row == 1
    out, _ = orc.create(np.array([[0, 2, 0], [-2, 4, 0]], np.int32), tensor_stride=[2, 2])
    assert out.shape == (2, 3)


def test_stride_worked_examples(orc):
    # tests/golden/stride_example.txt: S:87-88.
    for line in golden_lines("stride_example.txt"):
        lhs, rhs = line.split("->")
        cin, ts, cs = [x.strip() for x in lhs.split("|")]
        c = np.array([[int(x), 0] for x in cin.split(",")], np.int32)
        out = orc.stride(c, [int(cs)], [int(ts)])
        assert out[:, 0].tolist() == [int(x) for x in rhs.split(",")]


@pytest.mark.parametrize("sigma,ts", [(2, 1), (3, 2), (4, 4)])
def test_stride_brute_force(orc, sigma, ts):
    g = np.random.default_rng(sigma)
    c = g.integers(-40, 40, (800, 3)) * ts
    rows = np.concatenate([c, g.integers(0, 2, (800, 1))], axis=1).astype(np.int32)
    rows, _ = orc.create(rows, tensor_stride=[ts] * 3)
    out = orc.stride(rows, [sigma] * 3, [ts] * 3)
    s = ts * sigma
    seen, want = set(), []
    for r in rows.tolist():  # Python // is floor division: a separate implementation
        k = tuple(x // s * s for x in r[:3]) + (r[3],)
        if k not in seen:
            seen.add(k)
            want.append(k)
    assert out.tolist() == [list(k) for k in want]
    assert out.shape[0] <= rows.shape[0]


def test_labels_worked_examples(orc):
    # golden: S:78 (two points {2,2} -> 2, {2,5} -> IGNORE), P:181 reduction
    for line in golden_lines("labels_example.txt"):
        ign, rest = line.split("|")
        labs, want = rest.split("->")
        labs = np.array([int(v) for v in labs.split()], np.int32)
        pts = np.full((labs.shape[0], 3), 0.55, np.float32)  # all in one voxel
        coords, p2r, first = orc.quantize(pts, 0.1)
        assert coords.shape[0] == 1
        assert orc.labels(p2r, labs, 1, int(ign)).tolist() == [int(want)]


@pytest.mark.parametrize("seed", [0, 1])
def test_labels_brute_force(orc, seed):
    # brute force from the definition: a voxel keeps a label iff every point carries it
    g = np.random.default_rng(seed)
    pts = g.uniform(-1, 1, (4000, 3)).astype(np.float32)
    labs = g.integers(0, 3, 4000).astype(np.int32)
    # make some voxels label-pure on purpose
    coords, p2r, first = orc.quantize(pts, 0.25)
    pure = g.random(coords.shape[0]) < 0.5
    labs = np.where(pure[p2r], 9, labs).astype(np.int32)
    got = orc.labels(p2r, labs, coords.shape[0], -1)
    sets = {}
    for p, r in enumerate(p2r):
        sets.setdefault(int(r), set()).add(int(labs[p]))
    want = [next(iter(sets[r])) if len(sets[r]) == 1 else -1 for r in range(coords.shape[0])]
    assert got.tolist() == want
    assert (got == 9).sum() >= pure.sum() // 2  # the planted pure voxels survive


def test_labels_point_order_invariant(orc):
    # the reduction is a set function of the voxel's labels: permuting the points changes
    # the row numbering (first occurrence, R8) but not the label of any voxel
    g = np.random.default_rng(5)
    pts = g.uniform(0, 1, (3000, 3)).astype(np.float32)
    labs = g.integers(0, 2, 3000).astype(np.int32)
    c1, p1, _ = orc.quantize(pts, 0.2)
    l1 = orc.labels(p1, labs, c1.shape[0])
    perm = g.permutation(3000)
    c2, p2, _ = orc.quantize(pts[perm], 0.2)
    l2 = orc.labels(p2, labs[perm], c2.shape[0])
    d1 = {tuple(c): l for c, l in zip(c1.tolist(), l1.tolist())}
    d2 = {tuple(c): l for c, l in zip(c2.tolist(), l2.tolist())}
    assert d1 == d2


def test_expand_pins(orc):
    # f4 generative output coordinates: {u + i * s}.
    # (1) the region {0} is the identity (same rows, same order)
    g = np.random.default_rng(8)
    rows = np.concatenate([g.integers(-20, 20, (500, 3)) * 2, g.integers(0, 2, (500, 1))], axis=1).astype(np.int32)
    c, _ = orc.create(rows, [2, 2, 2])
    assert np.array_equal(orc.expand(c, np.zeros((1, 3), np.int32)), c)
    # (2) brute force: the set and the first-occurrence order of (row, offset)
    offs = orc.region(0, 3, [3, 3, 3])
    got = orc.expand(c, offs, [1, 1, 1])
    want, seen = [], set()
    for r in c.tolist():
        for o in offs.tolist():
            key = (r[0] + o[0], r[1] + o[1], r[2] + o[2], r[3])
            if key not in seen:
                seen.add(key)
                want.append(key)
    assert [tuple(x) for x in got.tolist()] == want
    # (3) upsampling: expanding the stride-2 set of a full grid by {0,1}^3 at the fine stride
    #     recovers exactly the full grid (as a set) — the generative transposed conv's output
    fine = full_grid(6, 3)
    coarse = orc.stride(fine, [2, 2, 2])
    up = orc.expand(coarse, orc.region(0, 3, [2, 2, 2]), [1, 1, 1])
    assert sorted(map(tuple, up.tolist())) == sorted(map(tuple, fine.tolist()))
    # (4) batch indices never move (R18)
    assert set(got[:, 3].tolist()) == set(c[:, 3].tolist())


def test_packed_key_domain(orc):
    # Reading R19 (the ABI domain of mk.h): D = 4 keeps t in [-2^15, 2^15) and b <= 65534;
    # D = 5..7 keeps axes 0-2 in [-2^19, 2^19), axes 3-5 in [-2^11, 2^11), axis 6 in
    # [-2^15, 2^15).  The first row outside the domain is reported with COORD_RANGE.
    r4 = np.zeros((10, 5), np.int32)
    r4[6, 3] = -32768            # the lowest representable t: accepted
    orc.create(r4.copy())
    for row, col, v in ((4, 3, 40000), (2, 3, -32769), (7, 4, 65535)):
        bad = r4.copy()
        bad[row, col] = v
        with pytest.raises(orc.OracleError) as e:
            orc.create(bad)
        assert e.value.status == orc.COORD_RANGE and e.value.row == row
    r7 = np.zeros((6, 8), np.int32)
    r7[1, 0], r7[2, 3], r7[3, 6] = (1 << 19) - 1, -(1 << 11), 32767  # edges: accepted
    orc.create(r7.copy())
    for row, col, v in ((3, 0, 1 << 19), (5, 4, 1 << 11), (1, 6, -32769)):
        bad = r7.copy()
        bad[row, col] = v
        with pytest.raises(orc.OracleError) as e:
            orc.create(bad)
        assert e.value.status == orc.COORD_RANGE and e.value.row == row
    # quantize applies the same domain to floor(p / v): t = 40000.5 / 1.0 -> 40000
    pts = np.zeros((5, 4), np.float32)
    pts[3, 3] = 40000.5
    with pytest.raises(orc.OracleError) as e:
        orc.quantize(pts, 1.0)
    assert e.value.status == orc.COORD_RANGE and e.value.row == 3
    # D <= 3: any int32 component
    big = np.array([[2**31 - 1, -2**31, 0, 0]], np.int32)
    assert np.array_equal(orc.create(big)[0], big)
