"""GPU <-> oracle parity of the integer path: coordinates, hash lookups and kernel maps
must be byte-identical (BASELINE.json north_star; DESIGN.md §3 R22)."""
import numpy as np
import pytest
import torch

import synthetic
from conftest import full_grid
from parity import Spec, csr_host, map_pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mk():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1904_08755_b200 as m
    return m


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t if dtype is None else t.to(dtype)


# ------------------------------------------------------------------ quantize / create
@pytest.mark.parametrize("seed,n,D,span,voxel", [(0, 1, 3, 1.0, 0.1), (1, 3000, 3, 1.0, 0.1), (2, 50000, 3, 3.0, 0.05),
                                                 (3, 20000, 2, 1.0, 0.01), (4, 7000, 1, 5.0, 0.3), (5, 40000, 4, 2.0, 0.25)])
def test_quantize_matches_oracle(mk, orc, seed, n, D, span, voxel):
    g = np.random.default_rng(seed)
    pts = g.uniform(-span, span, (n, D)).astype(np.float32)
    batch = g.integers(0, 4, n).astype(np.int32)
    c, p2r, first = mk.coords_quantize(dev(pts), voxel, dev(batch))
    oc, op2r, ofirst = orc.quantize(pts, voxel, batch)
    assert np.array_equal(c.export().cpu().numpy(), oc)
    assert np.array_equal(p2r.cpu().numpy(), op2r)
    assert np.array_equal(first.cpu().numpy(), ofirst)


def test_quantize_room_full_size(mk, orc):
    # cfg2 shape: ~1M raw points -> ~150k voxels at 2 cm (BASELINE configs[1])
    pts = synthetic.room_points(2001)
    c, p2r, first = mk.coords_quantize(dev(pts), synthetic.ROOM_VOXEL)
    oc, op2r, ofirst = orc.quantize(pts, synthetic.ROOM_VOXEL)
    assert np.array_equal(c.export().cpu().numpy(), oc)
    assert np.array_equal(p2r.cpu().numpy(), op2r)
    assert np.array_equal(first.cpu().numpy(), ofirst)


def test_quantize_worked_example_and_r6(mk):
    pts = np.array([[0.12, 0.34, 0.56], [0.3, 0.3, 0.3], [0.58, 0.58, 0.58]], np.float32)
    c, _, _ = mk.coords_quantize(dev(pts[:1]), 0.1)
    assert c.export().cpu().tolist() == [[1, 3, 5, 0]]
    c, _, _ = mk.coords_quantize(dev(pts[1:2]), 0.1)
    assert c.export().cpu().tolist() == [[3, 3, 3, 0]]  # R6: fp32 division
    c, _, _ = mk.coords_quantize(dev(pts[2:3]), 0.02)
    assert c.export().cpu().tolist() == [[29, 29, 29, 0]]


def test_quantize_errors(mk):
    pts = np.zeros((5000, 3), np.float32)
    pts[3001, 1] = np.nan
    pts[4000, 0] = np.inf
    with pytest.raises(mk.MkError) as e:
        mk.coords_quantize(dev(pts), 0.1)
    assert e.value.name == "MK_ERR_NONFINITE_INPUT" and e.value.row == 3001
    pts = np.zeros((100, 2), np.float32)
    pts[77, 0] = 3e9
    with pytest.raises(mk.MkError) as e:
        mk.coords_quantize(dev(pts), 1.0)
    assert e.value.name == "MK_ERR_COORD_RANGE" and e.value.row == 77
    b = np.zeros(100, np.int32)
    b[12] = -1
    with pytest.raises(mk.MkError) as e:
        mk.coords_quantize(dev(np.zeros((100, 3), np.float32)), 1.0, dev(b))
    assert e.value.name == "MK_ERR_INVALID_ARGUMENT" and e.value.row == 12


def test_empty_inputs(mk):
    c, p2r, first = mk.coords_quantize(torch.zeros((0, 3), device="cuda"), 0.1)
    assert c.n == 0 and p2r.numel() == 0
    m = mk.kmap_build(c, c, mk.Region(mk.HYPERCUBE, 3, 3))
    assert m.n_pairs == 0 and m.K == 27
    W = torch.randn(27, 16, 16, device="cuda")
    y = mk.conv_forward(m, torch.zeros((0, 16), device="cuda"), W)
    assert y.shape == (0, 16)


@pytest.mark.parametrize("D,ts", [(3, 1), (3, 2), (4, 1), (2, 3)])
def test_create_matches_oracle(mk, orc, D, ts):
    g = np.random.default_rng(D * 7 + ts)
    rows = np.concatenate([g.integers(-60, 60, (30000, D)) * ts, g.integers(0, 3, (30000, 1))], axis=1).astype(np.int32)
    c, inv = mk.coords_create(dev(rows), [ts] * D, return_inverse=True)
    oc, oinv = orc.create(rows, [ts] * D)
    assert np.array_equal(c.export().cpu().numpy(), oc)
    assert np.array_equal(inv.cpu().numpy(), oinv)
    assert c.tensor_stride == [ts] * D


def test_create_errors(mk):
    rows = np.zeros((300, 4), np.int32)
    rows[:, :3] = 2
    rows[123, 1] = 3
    with pytest.raises(mk.MkError) as e:
        mk.coords_create(dev(rows), [2, 2, 2])
    assert e.value.name == "MK_ERR_STRIDE" and e.value.row == 123
    r4 = np.zeros((10, 5), np.int32)
    r4[4, 3] = 40000  # t outside the packed 4D key domain
    with pytest.raises(mk.MkError) as e:
        mk.coords_create(dev(r4))
    assert e.value.name == "MK_ERR_COORD_RANGE" and e.value.row == 4


@pytest.mark.parametrize("sigma,ts,D", [(2, 1, 3), (2, 2, 3), (3, 1, 3), (2, 1, 4), (4, 1, 2)])
def test_stride_matches_oracle(mk, orc, sigma, ts, D):
    g = np.random.default_rng(sigma * 10 + ts)
    rows = np.concatenate([g.integers(-80, 80, (20000, D)) * ts, g.integers(0, 2, (20000, 1))], axis=1).astype(np.int32)
    c = mk.coords_create(dev(rows), [ts] * D)
    s = mk.coords_stride(c, [sigma] * D)
    oc, _ = orc.create(rows, [ts] * D)
    assert np.array_equal(s.export().cpu().numpy(), orc.stride(oc, [sigma] * D, [ts] * D))
    assert s.tensor_stride == [ts * sigma] * D


def test_lookup_matches_oracle(mk, orc):
    g = np.random.default_rng(9)
    rows = np.concatenate([g.integers(-30, 30, (20000, 3)), g.integers(0, 2, (20000, 1))], axis=1).astype(np.int32)
    q = np.concatenate([g.integers(-31, 31, (50000, 3)), g.integers(0, 3, (50000, 1))], axis=1).astype(np.int32)
    c = mk.coords_create(dev(rows))
    oc, _ = orc.create(rows)
    assert np.array_equal(c.lookup(dev(q)).cpu().numpy(), orc.lookup(oc, q))


@pytest.mark.parametrize("batches", [[0, 1, 2, 7, 9], [3, 5000]])
def test_per_batch_regions_match_oracle(mk, orc, batches):
    # >= 1.6M rows: the table gets per-batch regions (mk_internal.cuh TableRef); uneven
    # batch sizes, batch indices with no rows (lookups of them are absent), and a batch
    # index >= kMaxSub (4096), which falls back to the flat table.  Rows, lookups and a
    # 3x3x3 map are byte-identical to the oracle's.
    g = np.random.default_rng(sum(batches))
    sizes = g.dirichlet(np.ones(len(batches))) * 1_700_000 + 20_000
    parts = []
    for b, n in zip(batches, sizes.astype(int)):
        xyz = g.integers(-120, 120, (n, 3))
        parts.append(np.concatenate([xyz, np.full((n, 1), b)], axis=1))
    rows = np.concatenate(parts).astype(np.int32)
    c = mk.coords_create(dev(rows))
    oc, _ = orc.create(rows)
    assert np.array_equal(c.export().cpu().numpy(), oc)
    q = np.concatenate([g.integers(-121, 121, (200000, 3)), g.choice(batches + [4, 8, 4095], (200000, 1))],
                       axis=1).astype(np.int32)
    assert np.array_equal(c.lookup(dev(q)).cpu().numpy(), orc.lookup(oc, q))
    sel = np.isin(oc[:, 3], batches[:2])  # a map on a slice of the rows (oracle time)
    sub = np.ascontiguousarray(oc[sel][::8])
    cs = mk.coords_create(dev(sub))
    map_pair(mk, orc, c, cs, oc, sub, Spec(0, 3, 3), [1, 1, 1], what="regions map")


# ------------------------------------------------------------------ kernel maps
def _check_map(mk, orc, cin_np, cout_np, spec, scale, transposed, ci, co):
    """GPU map of the GPU coordinate handles vs the oracle's map of the oracle's coordinates
    and offsets (byte-identical); the region tables of both sides agree too."""
    assert np.array_equal(mk.region_offsets(spec.mk(mk)), spec.orc(orc))
    return map_pair(mk, orc, ci, co, cin_np, cout_np, spec, scale, transposed)[0]


@pytest.mark.parametrize("kind,D,size,dil", [(0, 3, 3, 1), (0, 3, 5, 1), (1, 3, 3, 1), (2, 4, 3, 1), (0, 4, 3, 1),
                                             (0, 3, 3, 2), (0, 3, 2, 1), (0, 2, 7, 1)])
def test_kmap_submanifold_matches_oracle(mk, orc, kind, D, size, dil):
    g = np.random.default_rng(kind * 100 + D * 10 + size)
    rows = np.concatenate([g.integers(-25, 25, (40000, D)), g.integers(0, 2, (40000, 1))], axis=1).astype(np.int32)
    c = mk.coords_create(dev(rows))
    oc, _ = orc.create(rows)
    _check_map(mk, orc, oc, oc, Spec(kind, D, size, dil), [1] * D, False, c, c)


def test_kmap_worked_examples(mk):
    c = mk.coords_create(dev(full_grid(4, 2)))
    assert mk.kmap_build(c, c, mk.Region(mk.HYPERCUBE, 2, 3)).n_pairs == 100
    c1 = mk.coords_create(dev(np.array([[5, 5, 5, 0]], np.int32)))
    m = mk.kmap_build(c1, c1, mk.Region(mk.HYPERCUBE, 3, 3))
    ptr, ins, outs = csr_host(m)
    assert m.n_pairs == 1 and ptr[14] - ptr[13] == 1  # one pair at offset 0


@pytest.mark.parametrize("K,ts", [(2, 1), (3, 1), (2, 2)])
def test_kmap_strided_and_transposed_match_oracle(mk, orc, K, ts):
    g = np.random.default_rng(K * 10 + ts)
    rows = np.concatenate([g.integers(-40, 40, (30000, 3)) * ts, g.integers(0, 2, (30000, 1))], axis=1).astype(np.int32)
    fine = mk.coords_create(dev(rows), [ts] * 3)
    coarse = mk.coords_stride(fine, [2, 2, 2])
    ofine, _ = orc.create(rows, [ts] * 3)
    ocoarse = orc.stride(ofine, [2, 2, 2], [ts] * 3)
    assert np.array_equal(coarse.export().cpu().numpy(), ocoarse)
    r = Spec(0, 3, K)
    m = _check_map(mk, orc, ofine, ocoarse, r, [ts] * 3, False, fine, coarse)
    if K == 2:
        assert m.n_pairs == fine.n  # R3 partition pin
    _check_map(mk, orc, ocoarse, ofine, r, [ts] * 3, True, coarse, fine)


def test_kmap_room_full_size(mk, orc):
    # BASELINE configs[1]: ScanNet-shaped room, 3x3x3, full size — maps bit-exact
    pts = synthetic.room_points(2002)
    c, _, _ = mk.coords_quantize(dev(pts), synthetic.ROOM_VOXEL)
    oc, _, _ = orc.quantize(pts, synthetic.ROOM_VOXEL)
    assert np.array_equal(c.export().cpu().numpy(), oc)
    _check_map(mk, orc, oc, oc, Spec(0, 3, 3), [1, 1, 1], False, c, c)


def test_kmap_video_hybrid_full_size(mk, orc):
    # BASELINE configs[2]: 3 frames x ~100k voxels, hybrid kernel (29 offsets)
    pts, fr = synthetic.video_points(3001)
    c3, _, _ = mk.coords_quantize(dev(pts), synthetic.VIDEO_VOXEL, dev(fr))
    rows4 = c3.export()
    rows4 = torch.cat([rows4[:, :3], rows4[:, 3:4], torch.zeros_like(rows4[:, :1])], dim=1)  # frame -> t, b = 0
    c4 = mk.coords_create(rows4)
    o3, _, _ = orc.quantize(pts, synthetic.VIDEO_VOXEL, fr)
    o4 = np.concatenate([o3, np.zeros((o3.shape[0], 1), np.int32)], axis=1)
    assert np.array_equal(c4.export().cpu().numpy(), o4)
    m = _check_map(mk, orc, o4, o4, Spec(2, 4, 3), [1] * 4, False, c4, c4)
    assert m.K == 29


@pytest.mark.parametrize("ignore", [-1, 255])
def test_labels_room_full_size(mk, orc, ignore):
    # BASELINE configs[1] scan with per-point labels that disagree inside some voxels
    # (label = coarse 6 cm cell parity of x + y, so voxels straddling a boundary mix labels;
    # plus 2% random label noise); bit-exact against the oracle's reduction.
    pts = synthetic.room_points(2004)
    g = np.random.default_rng(4)
    labs = (np.floor(pts[:, 0] / 0.06).astype(np.int64) + np.floor(pts[:, 1] / 0.06).astype(np.int64)) % 2
    labs = np.where(g.random(labs.shape[0]) < 0.02, 7, labs).astype(np.int32)
    c, p2r, first = mk.coords_quantize(dev(pts), synthetic.ROOM_VOXEL)
    got = mk.coords_labels(p2r, first, dev(labs), ignore_label=ignore).cpu().numpy()
    oc, op2r, ofirst = orc.quantize(pts, synthetic.ROOM_VOXEL)
    assert np.array_equal(p2r.cpu().numpy(), op2r)
    want = orc.labels(op2r, labs, oc.shape[0], ignore)
    assert np.array_equal(got, want)
    assert 0 < (want == ignore).sum() < want.shape[0]  # both outcomes occur


def test_labels_empty(mk):
    c, p2r, first = mk.coords_quantize(torch.zeros((0, 3), device="cuda"), 0.1)
    out = mk.coords_labels(p2r, first, torch.zeros(0, dtype=torch.int32, device="cuda"))
    assert out.numel() == 0


@pytest.mark.parametrize("K", [2, 3])
def test_expand_and_generative_transposed_conv(mk, orc, K):
    # f4: generative output coordinates {u + i * s_f} of a stride-2 set, byte-identical
    # to the oracle, then the transposed conv onto them against the fp64 oracle.
    from gpu_util import FP32_TOL, assert_close
    g = np.random.default_rng(40 + K)
    rows = np.concatenate([g.integers(-40, 40, (20000, 3)), g.integers(0, 2, (20000, 1))], axis=1).astype(np.int32)
    oc, _ = orc.create(rows)
    fine = mk.coords_create(dev(rows))
    coarse = mk.coords_stride(fine, [2, 2, 2])
    spec = Spec(0, 3, K)
    region = spec.mk(mk)
    up = mk.coords_expand(coarse, region, [1, 1, 1])
    ocoarse = orc.stride(oc, [2, 2, 2])
    oup = orc.expand(ocoarse, spec.orc(orc), [1, 1, 1])
    assert np.array_equal(up.export().cpu().numpy(), oup)
    assert up.tensor_stride == [1, 1, 1]
    m, okm = map_pair(mk, orc, coarse, up, ocoarse, oup, spec, [1, 1, 1], transposed=True)
    Y = g.standard_normal((coarse.n, 32)).astype(np.float32)
    W = (g.standard_normal((m.K, 16, 32)) * 0.1).astype(np.float32)
    z = mk.conv_transpose_forward(m, dev(Y), dev(W)).cpu().numpy()
    z64 = orc.conv_forward(okm, Y, W, up.n)
    assert_close(z, z64, orc.conv_forward(okm, np.abs(Y), np.abs(W), up.n), FP32_TOL, "generative convT")
    with pytest.raises(mk.MkError) as e:  # the output stride must divide the input stride
        mk.coords_expand(coarse, region, [3, 3, 3])
    assert e.value.name == "MK_ERR_STRIDE"


def test_deferred_quantize_matches_eager(mk):
    # mk_coords_quantize_deferred: same rows, maps and kernel map as the eager call; the count
    # is collected by the kernel-map build (or Coords.n)
    pts = torch.from_numpy(synthetic.room_points(2000)).cuda()
    c0, p0, f0 = mk.coords_quantize(pts, synthetic.ROOM_VOXEL)
    c1, p1, f1 = mk.coords_quantize(pts, synthetic.ROOM_VOXEL, deferred=True)
    assert f1.shape[0] == pts.shape[0]  # full capacity
    m1 = mk.kmap_build(c1, c1, mk.Region(mk.HYPERCUBE, 3, 3))  # resolves the count
    assert c1.n == c0.n
    assert torch.equal(c1.export(), c0.export())
    assert torch.equal(p1, p0) and torch.equal(f1[: c1.n], f0)
    m0 = mk.kmap_build(c0, c0, mk.Region(mk.HYPERCUBE, 3, 3))
    for a, b in zip(mk.kmap_export(m1), mk.kmap_export(m0)):
        assert torch.equal(a, b)


def test_deferred_quantize_reports_errors_at_first_use(mk):
    pts = torch.rand((500, 3), device="cuda")
    pts[137, 1] = float("nan")
    c = mk.coords_quantize(pts, 0.1, return_maps=False, deferred=True)  # enqueued, no wait
    with pytest.raises(mk.MkError) as e:
        _ = c.n
    assert e.value.name == "MK_ERR_NONFINITE_INPUT" and e.value.row == 137
    with pytest.raises(mk.MkError):
        mk.kmap_build(c, c, mk.Region(mk.HYPERCUBE, 3, 3))


def test_deferred_quantize_mailbox_slot_reuse(mk):
    # more pending handles than mailbox slots (1024): the oldest ones find their slot reused
    # and fall back to the device words once their build event has completed
    g = np.random.default_rng(9)
    pts = [torch.from_numpy(g.random((200 + i % 7, 3)).astype(np.float32)).cuda() for i in range(8)]
    want = [mk.coords_quantize(p, 0.05, return_maps=False).n for p in pts]
    hs = [mk.coords_quantize(pts[i % 8], 0.05, return_maps=False, deferred=True) for i in range(1100)]
    torch.cuda.synchronize()
    assert [h.n for h in hs] == [want[i % 8] for i in range(1100)]
