"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded
inputs.  Integer / index stages must be bit-exact; kNN on float data follows the tolerance
rule of tests/knn_check.py; kNN on integer data (F16_EXACT) must be bit-exact.
"""
import numpy as np
import pytest
import torch

from paper_2605_10135_b200 import datagen
from tests.knn_check import check_knn

pytestmark = pytest.mark.gpu
SENT = 0xFFFFFFFF


@pytest.fixture(scope="module")
def api():
    from paper_2605_10135_b200 import api as a
    a.load()
    return a


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def _clustered(n, d, seed, integer=False):
    x = datagen.mixture(n, d, 0.5, seed=seed)
    if integer:
        x = torch.clamp(torch.round(40 * torch.clamp_min(x + 0.5, 0)), 0, 255)
    return x


# ------------------------------------------------------------------ GEMM core (step 4b)
@pytest.mark.parametrize("prec", [1, 2])
def test_gemm_probe_matches_matmul(api, prec):
    xa = datagen.sift_like(300, 128, seed=1)
    xb = datagen.sift_like(260, 128, seed=2)
    if prec == 2:
        xa, xb = datagen.gaussian(300, 128, seed=1), datagen.gaussian(260, 128, seed=2)
    # the augmented operands make the accumulator the selection key |b_j|^2 - 2 a_i.b_j
    out = api.scalegann_gemm_probe(xa.cuda(), xb.cuda(), precision=prec).cpu()
    ref = (xb.double() ** 2).sum(1)[None, :] - 2 * (xa.double() @ xb.double().T)
    if prec == 1:   # integer data on kind::f16 with fp32 accumulation: exact
        assert torch.equal(out.double(), ref)
    else:
        assert torch.allclose(out.double(), ref, rtol=0, atol=5e-2 * ref.abs().max().item() ** 0.5)


# ------------------------------------------------------------------ a5 kNN
@pytest.mark.parametrize("m,L", [(1000, 64), (1300, 128), (129, 128), (65, 64), (40, 64), (2, 8), (2600, 256),
                                 (300, 256)])
def test_knn_integer_exact(api, oracle_mod, m, L):
    x = datagen.sift_like(m, 128, seed=m)
    ids, dd = api.scalegann_knn(x.cuda(), L)
    oi, od = oracle_mod.knn(x.numpy(), L)
    assert np.array_equal(u32(ids), oi)
    assert np.array_equal(dd.cpu().numpy(), od)


def test_knn_u8_exact(api, oracle_mod):
    x = datagen.sift_like(1500, 128, seed=7, as_u8=True)
    ids, dd = api.scalegann_knn(x.cuda(), 128)
    oi, od = oracle_mod.knn(x.numpy(), 128)
    assert np.array_equal(u32(ids), oi) and np.array_equal(dd.cpu().numpy(), od)


@pytest.mark.parametrize("d", [128, 96, 100])
def test_knn_float_tolerance(api, oracle_mod, d):
    x = datagen.gaussian(2000, d, seed=d)
    ids, dd = api.scalegann_knn(x.cuda(), 64)
    oi, od = oracle_mod.knn(x.numpy(), 64)
    fails, msg = check_knn(u32(ids), dd.cpu().numpy(), oi, od, x.numpy())
    assert fails == 0, msg


def test_knn_subset_and_queries(api, oracle_mod):
    x = datagen.sift_like(3000, 128, seed=11)
    idm = torch.arange(5, 3000, 3, dtype=torch.int32)
    ids, dd = api.scalegann_knn(x.cuda(), 32, ida=idm.cuda())
    oi, od = oracle_mod.knn(x.numpy(), 32, ida=idm.numpy().astype(np.uint32))
    assert np.array_equal(u32(ids), oi) and np.array_equal(dd.cpu().numpy(), od)
    q = datagen.sift_like(200, 128, seed=12)
    gi, gd = api.scalegann_knn(q.cuda(), 10, xb=x.cuda(), self_exclude=False)
    oi, od = oracle_mod.knn(q.numpy(), 10, xb=x.numpy(), self_exclude=False)
    assert np.array_equal(u32(gi), oi) and np.array_equal(gd.cpu().numpy(), od)


def test_knn_inner_product(api, oracle_mod):
    x = datagen.sift_like(700, 128, seed=13)
    ids, dd = api.scalegann_knn(x.cuda(), 16, metric=1)
    oi, od = oracle_mod.knn(x.numpy(), 16, metric=1)
    assert np.array_equal(u32(ids), oi) and np.array_equal(dd.cpu().numpy(), od)


def test_knn_duplicates_ties(api, oracle_mod):
    x = datagen.sift_like(400, 128, seed=14)
    x[200:300] = x[100:200]          # exact duplicate rows: ties broken by id
    ids, dd = api.scalegann_knn(x.cuda(), 64)
    oi, od = oracle_mod.knn(x.numpy(), 64)
    assert np.array_equal(u32(ids), oi) and np.array_equal(dd.cpu().numpy(), od)


# ------------------------------------------------------------------ a6/a7 fed the oracle's kNN
@pytest.mark.parametrize("L,R", [(64, 32), (128, 64), (16, 16)])
def test_prune_reverse_bit_exact(api, oracle_mod, L, R):
    x = _clustered(2500, 32, seed=L + R)
    oi, od = oracle_mod.knn(x.numpy(), L)
    for rule in (0, 1):
        gp, gpd = api.scalegann_prune(torch.from_numpy(oi.view(np.int32)).cuda(), torch.from_numpy(od).cuda(), R,
                                      rule=rule)
        op, opd = oracle_mod.prune(oi, od, R, rule=rule)
        assert np.array_equal(u32(gp), op)
        assert np.array_equal(gpd.cpu().numpy(), opd)
    gf, gfd = api.scalegann_reverse(torch.from_numpy(op.view(np.int32)).cuda(), torch.from_numpy(opd).cuda())
    of, ofd = oracle_mod.reverse(op, opd)
    assert np.array_equal(u32(gf), of)
    assert np.array_equal(gfd.cpu().numpy(), ofd)


def test_reverse_hub_rows(api, oracle_mod):
    # a hub with in-degree >> 256 exercises the chunked segment sort
    m, R = 2000, 8
    rng = np.random.default_rng(3)
    pr = np.stack([rng.permutation(m)[:R] for _ in range(m)]).astype(np.uint32)
    pr[:, 0] = 7
    pr[7, 0] = 8
    for i in range(m):  # keep rows free of duplicates / self
        row = [v for v in pr[i] if v != i]
        while len(set(row)) < R:
            row = list(dict.fromkeys(row + [int(rng.integers(m))]))
            row = [v for v in row if v != i]
        pr[i] = np.array(row[:R], np.uint32)
    prd = rng.random((m, R)).astype(np.float32)
    gf, gfd = api.scalegann_reverse(torch.from_numpy(pr.view(np.int32)).cuda(), torch.from_numpy(prd).cuda())
    of, ofd = oracle_mod.reverse(pr, prd)
    assert np.array_equal(u32(gf), of) and np.array_equal(gfd.cpu().numpy(), ofd)


# ------------------------------------------------------------------ a2/a3 partition
@pytest.mark.parametrize("block,kind", [(65536, "gauss"), (1024, "gauss"), (997, "clustered"), (256, "sift")])
def test_partition_bit_exact(api, oracle_mod, block, kind):
    n = 10_000
    if kind == "gauss":
        x, k = datagen.gaussian(n, 128), 2
    elif kind == "sift":
        x, k = datagen.sift_like(n, 128, seed=5), 8
    else:
        x, k = _clustered(n, 64, seed=6), 8
    C = x[:: n // k][:k].clone().contiguous()
    home, pd, counts = api.scalegann_partition(x.cuda(), C.cuda(), omega=2, block_size=block)
    r = oracle_mod.partition(x.numpy(), C.numpy(), omega=2, block_size=block)
    assert np.array_equal(u32(home), r["home"])
    assert np.array_equal(pd.cpu().numpy(), r["primary_d"])
    assert counts["sizes"] == r["sizes"].tolist() and counts["repl"] == r["repl"].tolist()


@pytest.mark.parametrize("eps", [1.0, 1.05, 1.1, 1.5, 3.0])
def test_partition_epsilon_sweep_bit_exact(api, oracle_mod, eps):
    """§8(f) NEXT-2: the eps values of the paper's selectivity sweep, GPU == oracle,
    and eps <= 1 places no replica (d' < eps * d is impossible for d' >= d)."""
    n, k = 10_000, 8
    x = datagen.sift_like(n, 128, seed=7)
    C = x[:: n // k][:k].clone().contiguous()
    home, pd, counts = api.scalegann_partition(x.cuda(), C.cuda(), omega=2, epsilon=eps, block_size=1024)
    r = oracle_mod.partition(x.numpy(), C.numpy(), omega=2, eps=eps, block_size=1024)
    assert np.array_equal(u32(home), r["home"])
    assert counts["repl"] == r["repl"].tolist()
    if eps <= 1.0:
        assert sum(counts["repl"]) == 0


def test_partition_capacity_binding_and_omega3(api, oracle_mod):
    x = _clustered(6000, 16, seed=9)
    C = x[:6].clone()                      # poor centroids -> capacity binds
    for omega, cap in ((3, 0), (2, 1700)):
        home, pd, counts = api.scalegann_partition(x.cuda(), C.cuda(), omega=omega, epsilon=1.5, block_size=500,
                                                   capacity=cap)
        r = oracle_mod.partition(x.numpy(), C.numpy(), omega=omega, eps=1.5, block_size=500, capacity=cap)
        assert np.array_equal(u32(home), r["home"])


def test_idmap_and_inv(api, oracle_mod):
    x = datagen.gaussian(5000, 16)
    C = x[:3].clone()
    home, pd, counts = api.scalegann_partition(x.cuda(), C.cuda(), omega=2, epsilon=1.5)
    inv = torch.full((5000, 2), -1, dtype=torch.int32, device="cuda")
    for s in range(3):
        idm = api.scalegann_shard_idmap(home, s, inv=inv)
        ref = oracle_mod.idmap(u32(home), s)
        assert np.array_equal(u32(idm), ref)
    hv, iv = u32(home), u32(inv)
    for g in range(0, 5000, 7):
        for h in range(2):
            if hv[g, h] != SENT:
                assert oracle_mod.idmap(hv, hv[g, h])[iv[g, h]] == g


# ------------------------------------------------------------------ a8 merge fed the oracle's shard graphs
def test_merge_bit_exact(api, oracle_mod):
    x = datagen.sift_like(6000, 32, seed=21)
    C = x[::2000][:3].clone()
    r = oracle_mod.partition(x.numpy(), C.numpy(), omega=3, eps=1.6)
    home = torch.from_numpy(r["home"].view(np.int32)).cuda()
    idm_g, g_g, gd_g, idm_o, g_o, gd_o = [], [], [], [], [], []
    for s in range(3):
        im = oracle_mod.idmap(r["home"], s)
        ids, dd = oracle_mod.knn(x.numpy(), 16, ida=im)
        pr, prd = oracle_mod.prune(ids, dd, 8)
        f, fd = oracle_mod.reverse(pr, prd)
        idm_o.append(im), g_o.append(f), gd_o.append(fd)
        idm_g.append(api.scalegann_shard_idmap(home, s))
        g_g.append(torch.from_numpy(f.view(np.int32)).cuda())
        gd_g.append(torch.from_numpy(fd).cuda())
    m, md = api.scalegann_merge(home, idm_g, g_g, gd_g)
    om, omd = oracle_mod.merge(r["home"], idm_o, g_o, gd_o)
    assert np.array_equal(u32(m), om) and np.array_equal(md.cpu().numpy(), omd)


@pytest.mark.parametrize("world", [2, 3])
def test_merge_emulated_ranks_equal_single(api, world):
    """The distributed streaming protocol (plan -> fold shards -> records -> exchange -> fold
    records), with `world` ranks emulated in one process, gives owner rows that reassemble to the
    single-process merged graph byte for byte."""
    from paper_2605_10135_b200.pipeline import BuildConfig, build_index, lpt_owner
    x = datagen.sift_like(8000, 64, seed=31).cuda()
    cfg = BuildConfig(k=4, omega=3, epsilon=1.5, L=32, R=16)
    idx = build_index(x, cfg)
    home, n = idx.home, x.shape[0]
    sizes = idx.sizes
    idm, gs, gds = [], [], []
    for s in range(4):
        idm.append(api.scalegann_shard_idmap(home, s))
        g, gd = api.scalegann_build_shard(x, idm[-1], cfg.L, cfg.R)
        gs.append(g), gds.append(gd)
    owner = lpt_owner(sizes, world)
    W = 2 + 2 * cfg.R
    st = {}
    for rk in range(world):
        oi, rs, send, recv, no = api.scalegann_merge_plan(home, owner, rk, world)
        m, md = api.scalegann_merge_init(no, cfg.R)
        sendbuf = torch.empty(max(sum(send), 1) * W, dtype=torch.int32, device="cuda")
        for s in range(4):
            if owner[s] == rk:
                api.scalegann_merge_shard(home, owner, rk, world, s, idm[s], gs[s], gds[s], oi, rs, m, md, sendbuf)
        chunks = list(torch.split(sendbuf[: sum(send) * W], [c * W for c in send]))
        st[rk] = (oi, m, md, chunks, send, recv)
    full = torch.full_like(idx.merged, -1)
    full_d = torch.full_like(idx.merged_d, float("nan"))
    for rk in range(world):
        oi, m, md, _, _, recv = st[rk]
        recvbuf = torch.cat([st[src][3][rk] for src in range(world)])
        assert recvbuf.numel() == sum(recv) * W
        api.scalegann_merge_finish(cfg.omega, oi, recvbuf, sum(recv), m, md)
        own = torch.tensor(owner, device="cuda")[home[:, 0].long()] == rk
        full[own], full_d[own] = m, md
    assert torch.equal(full, idx.merged) and torch.equal(full_d, idx.merged_d)


# ------------------------------------------------------------------ a9 search
def test_search_matches_oracle(api, oracle_mod):
    x = datagen.sift_like(3000, 32, seed=41)
    ids, dd = oracle_mod.knn(x.numpy(), 16)
    q = datagen.sift_like(100, 32, seed=42)
    out, gt, rec = api.scalegann_search_eval(x.cuda(), torch.from_numpy(ids.view(np.int32)).cuda(), 0, q.cuda(),
                                             topk=10, beam=32)
    oo, _, _ = oracle_mod.search(x.numpy(), ids, 0, q.numpy(), topk=10, beam=32)
    assert np.array_equal(u32(out), oo)
    ogt, _ = oracle_mod.knn(q.numpy(), 10, xb=x.numpy(), self_exclude=False)
    assert np.array_equal(u32(gt), ogt)
    assert abs(rec - oracle_mod.recall(oo, ogt)) < 1e-12


@pytest.mark.parametrize("d", [128, 40])
def test_search_u8_matches_oracle(api, oracle_mod, d):
    """u8 rows (BIGANN-shaped): the 16-byte load path (d = 128) and the scalar path (d = 40)
    give the oracle's result lists."""
    x = datagen.sift_like(3000, d, seed=45, as_u8=True)
    ids, _ = oracle_mod.knn(x.numpy(), 16)
    q = datagen.sift_like(100, d, seed=46, as_u8=True)
    out, gt, rec = api.scalegann_search_eval(x.cuda(), torch.from_numpy(ids.view(np.int32)).cuda(), 0, q.cuda(),
                                             topk=10, beam=32)
    oo, _, _ = oracle_mod.search(x.numpy(), ids, 0, q.numpy(), topk=10, beam=32)
    assert np.array_equal(u32(out), oo)


@pytest.mark.parametrize("kind,d", [("gauss", 128), ("deep", 96), ("gauss", 25), ("u8", 25), ("u8", 99)])
def test_search_exact_distances_match_oracle(api, oracle_mod, kind, d):
    """P8 with exact distances on the GPU too (f32: fp64 sum of squared differences, one f32
    rounding; u8: integers): result lists AND the distance-count proxy equal the
    oracle's, on float data and on odd widths (unaligned rows)."""
    if kind == "u8":
        x, q = datagen.sift_like(2500, d, seed=71, as_u8=True), datagen.sift_like(80, d, seed=72, as_u8=True)
    elif kind == "deep":
        x, q = datagen.mixture(2500, d, 0.7, seed=71, normalise=True), datagen.mixture(80, d, 0.7, seed=72, normalise=True)
    else:
        x, q = datagen.gaussian(2500, d, seed=71), datagen.gaussian(80, d, seed=72)
    ids, _ = oracle_mod.knn(x.numpy(), 16)
    g = torch.from_numpy(ids.view(np.int32)).cuda()
    out, _, _, nd = api.scalegann_search_eval(x.cuda(), g, 7, q.cuda(), topk=10, beam=24, return_ndist=True)
    oo, od, ond = oracle_mod.search(x.numpy(), ids, 7, q.numpy(), topk=10, beam=24)
    assert np.array_equal(u32(out), oo)
    assert nd == int(ond.sum())


def test_search_hash_visited_set_matches_oracle(api, oracle_mod):
    """n = 70,000 with beam 16, R = 8: the visited set is the per-query hash set (1,024 slots
    instead of a 2,188-word bitmap); the lists equal the oracle's."""
    x = datagen.sift_like(70_000, 8, seed=73)
    ids, _ = oracle_mod.knn(x.numpy(), 8)
    q = datagen.sift_like(64, 8, seed=74)
    out, _, _, nd = api.scalegann_search_eval(x.cuda(), torch.from_numpy(ids.view(np.int32)).cuda(), 0, q.cuda(),
                                              topk=10, beam=16, return_ndist=True)
    oo, _, ond = oracle_mod.search(x.numpy(), ids, 0, q.numpy(), topk=10, beam=16)
    assert np.array_equal(u32(out), oo)
    assert nd == int(ond.sum())


def test_search_validation(api):
    x = datagen.sift_like(500, 16, seed=75).cuda()
    g = torch.zeros(500, 8, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        api.scalegann_search_eval(x, g, 0, torch.zeros(4, 16, dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):
        api.scalegann_search_eval(x, g, 0, torch.zeros(4, 16))


def test_search_shards_split_only_matches_oracle(api, oracle_mod):
    """Split-only build (k = 3, omega = 1) searched per shard with result merge (P:432-470,
    reading R15): GPU == oracle list for list; per-shard search beats one global beam."""
    from paper_2605_10135_b200.pipeline import BuildConfig, build_index
    x = datagen.sift_like(6000, 64, seed=43)
    idx = build_index(x.cuda(), BuildConfig(k=3, omega=1, epsilon=1.0, L=32, R=16, block_size=1024))
    _, entries = api.scalegann_entry_points(idx.home, idx.primary_d, idx.sizes)
    q = datagen.sift_like(200, 64, seed=44)
    out, gt, rec = api.scalegann_search_eval_shards(x.cuda(), idx.merged, entries, q.cuda(), topk=10, beam=32)
    oo = oracle_mod.search_shards(x.numpy(), u32(idx.merged), entries, q.numpy(), topk=10, beam=32)
    assert np.array_equal(u32(out), oo)
    ogt, _ = oracle_mod.knn(q.numpy(), 10, xb=x.numpy(), self_exclude=False)
    assert np.array_equal(u32(gt), ogt)
    assert abs(rec - oracle_mod.recall(oo, ogt)) < 1e-12
    _, _, rec1 = api.scalegann_search_eval(x.cuda(), idx.merged, idx.entry, q.cuda(), topk=10, beam=32, gt=gt)
    assert rec > rec1
    # an empty shard's SENTINEL entry (scalegann_entry_points) is skipped, not an error
    out2, _, _ = api.scalegann_search_eval_shards(x.cuda(), idx.merged, list(entries) + [SENT], q.cuda(), topk=10,
                                                  beam=32, gt=gt)
    assert torch.equal(out2, out)


# ------------------------------------------------------------------ a1 k-means
def test_kmeans_distortion_within_1pct(api, oracle_mod):
    x = datagen.sift_like(50_000, 128, seed=51)
    C = api.scalegann_kmeans(x.cuda(), 8).cpu().numpy()
    _, od = oracle_mod.kmeans(x.numpy(), 8)
    assert oracle_mod.kmeans_distortion(x.numpy(), C) <= 1.01 * od


# ------------------------------------------------------------------ end to end (C0-sized)
@pytest.mark.parametrize("k,omega,eps", [(2, 2, 1.2), (3, 1, 1.0), (3, 2, 3.0)])
def test_end_to_end_integer_bit_exact(api, oracle_mod, k, omega, eps):
    """SIFT-shaped integer data: every stage is exact, so the GPU merged graph equals the
    oracle-built graph bit for bit (same centroids fed to both).  (3, 1, 1.0) is the split-only
    build of P:432-470 (no replicas); (3, 2, 3.0) the most selective-replication-heavy end of
    the eps sweep (§8(f) NEXT-2)."""
    from paper_2605_10135_b200.pipeline import BuildConfig, build_index
    x = datagen.sift_like(6000, 128, seed=61)
    cfg = BuildConfig(k=k, omega=omega, epsilon=eps, L=64, R=32, block_size=1024)
    idx = build_index(x.cuda(), cfg)
    C = idx.centroids.cpu().numpy()
    r = oracle_mod.partition(x.numpy(), C, omega=omega, eps=eps, block_size=1024)
    assert np.array_equal(u32(idx.home), r["home"])
    if omega == 1:
        assert int(r["repl"].sum()) == 0
    idm, gs, gds = [], [], []
    for s in range(k):
        im = oracle_mod.idmap(r["home"], s)
        ids, dd = oracle_mod.knn(x.numpy(), 64, ida=im)
        pr, prd = oracle_mod.prune(ids, dd, 32)
        f, fd = oracle_mod.reverse(pr, prd)
        idm.append(im), gs.append(f), gds.append(fd)
    om, omd = oracle_mod.merge(r["home"], idm, gs, gds)
    assert np.array_equal(u32(idx.merged), om)
    assert np.array_equal(idx.merged_d.cpu().numpy(), omd)
    ge, _ = oracle_mod.entry_points(r["home"], r["primary_d"], r["sizes"])
    assert idx.entry == ge


def test_end_to_end_c0_recall(api, oracle_mod):
    """C0 (10K x 128 Gaussian f32, 2 shards, R=32, L=64): recall@10 of the GPU-built merged
    graph within 0.5 points of the oracle-built graph (north_star criterion)."""
    from paper_2605_10135_b200.pipeline import BuildConfig, build_index
    w = datagen.C0
    x = w.data()
    q = w.queries()[:300]
    cfg = BuildConfig(k=w.k, L=w.L, R=w.R)
    idx = build_index(x.cuda(), cfg)
    C = idx.centroids.cpu().numpy()
    r = oracle_mod.partition(x.numpy(), C, omega=2)
    assert np.array_equal(u32(idx.home), r["home"])
    idm, gs, gds = [], [], []
    for s in range(w.k):
        im = oracle_mod.idmap(r["home"], s)
        ids, dd = oracle_mod.knn(x.numpy(), w.L, ida=im)
        pr, prd = oracle_mod.prune(ids, dd, w.R)
        f, fd = oracle_mod.reverse(pr, prd)
        idm.append(im), gs.append(f), gds.append(fd)
    om, _ = oracle_mod.merge(r["home"], idm, gs, gds)
    ge, _ = oracle_mod.entry_points(r["home"], r["primary_d"], r["sizes"])
    gt, _ = oracle_mod.knn(q.numpy(), 10, xb=x.numpy(), self_exclude=False)
    res_o, _, _ = oracle_mod.search(x.numpy(), om, ge, q.numpy(), topk=10, beam=64)
    res_g, _, _ = oracle_mod.search(x.numpy(), u32(idx.merged), idx.entry, q.numpy(), topk=10, beam=64)
    ro, rg = oracle_mod.recall(res_o, gt), oracle_mod.recall(res_g, gt)
    assert abs(ro - rg) <= 0.005, (ro, rg)


# ------------------------------------------------------------------ a5 wide rows (streamed-A kernel)
@pytest.mark.parametrize("d", [512, 300])
def test_knn_wide_integer_exact(api, oracle_mod, d):
    """d * 2 bytes beyond 4 resident atoms: both operands stream through the ring; integer data
    with 2 d max^2 < 2^24 stays F16_EXACT, so ids and dists are bit-identical to the oracle."""
    x = torch.clamp(torch.round(datagen.sift_like(1400, d, seed=d) / 4), 0, 60)
    ids, dd = api.scalegann_knn(x.cuda(), 64)
    oi, od = oracle_mod.knn(x.numpy(), 64)
    assert np.array_equal(u32(ids), oi) and np.array_equal(dd.cpu().numpy(), od)


def test_knn_c3_text_embedding_768(api, oracle_mod):
    """C3-shaped rows (768-d, power-law spectrum, L2-normalised): TF32 operands,
    fp32 accumulation, judged by the P4 tolerance rule."""
    x = datagen.mixture(1200, 768, 1.0, seed=31, normalise=True)
    ids, dd = api.scalegann_knn(x.cuda(), 64)
    oi, od = oracle_mod.knn(x.numpy(), 64)
    fails, msg = check_knn(u32(ids), dd.cpu().numpy(), oi, od, x.numpy())
    assert fails == 0, msg


def test_knn_c2_deep_96(api, oracle_mod):
    """C2-shaped rows (96-d, spectrum beta 0.7, L2-normalised): TF32, tolerance rule."""
    x = datagen.mixture(2000, 96, 0.7, seed=32, normalise=True)
    ids, dd = api.scalegann_knn(x.cuda(), 128)
    oi, od = oracle_mod.knn(x.numpy(), 128)
    fails, msg = check_knn(u32(ids), dd.cpu().numpy(), oi, od, x.numpy())
    assert fails == 0, msg
