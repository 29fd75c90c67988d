"""Pins for the CPU oracle (oracle/oracle.c) against what the paper and the
mathematics fix — NOT against itself.  Each test names the passage or the
closed form it checks.  These run with -m "not gpu" in a few seconds.
"""
import ctypes
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SENT = 0xFFFFFFFF


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- P1 ----
def test_p1_small_integers_exact(oracle_mod):
    # integer data: every fmaf step is exact, so d^2 is the textbook integer
    x = np.array([[1, 2, 3], [0, 0, 0], [4, 0, 1]], np.float32)
    C = np.array([[0, 0, 0], [1, 1, 1]], np.float32)
    d = oracle_mod.centroid_dist(x, C)
    assert d.tolist() == [[14, 5], [0, 3], [17, 10]]


def test_p1_u8_promoted_exactly(oracle_mod):
    rng = np.random.default_rng(1)
    x = rng.integers(0, 256, (50, 128)).astype(np.uint8)
    C = rng.integers(0, 256, (3, 128)).astype(np.float32)
    d = oracle_mod.centroid_dist(x, C)
    ref = ((x.astype(np.int64)[:, None, :] - C.astype(np.int64)[None]) ** 2).sum(-1)  # < 2^24: exact
    assert np.array_equal(d, ref.astype(np.float32))


def test_p1_fma_chain_order(oracle_mod):
    # a case where fused vs unfused accumulation differ: fixes the stated fmaf order
    x = np.array([[1.0 + 2.0 ** -12, 1.0]], np.float32)
    C = np.zeros((1, 2), np.float32)
    acc = np.float32(0)
    for v in x[0]:
        acc = np.float32(np.float64(v) * np.float64(v) + np.float64(acc))  # exact fma then RN
    assert oracle_mod.centroid_dist(x, C)[0, 0] == acc


# ---------------------------------------------------------------- P2/P3 ----
def test_capacity_reading_r9(oracle_mod):
    # R9: cap = ceil(1.15 * ceil(n / (k (1 - theta0)))), theta0 = 0.4; values worked by hand:
    # C0 10000/(2*0.6) = 8333.3 -> 8334 -> 9584.1 -> 9585, C1 416666.7 -> 416667 -> 479168, ...
    assert oracle_mod.capacity(10_000, 2) == 9585
    assert oracle_mod.capacity(1_000_000, 4) == 479_168
    assert oracle_mod.capacity(10_000_000, 8) == 2_395_835
    assert oracle_mod.capacity(5_000_000, 8) == 1_197_918
    assert oracle_mod.capacity(100_000_000, 8) == 23_958_335
    # the property the reading exists for: with every replica budget at its
    # cap theta0*cap, the clusters still hold 1.15 n originals
    for n, k in ((10_000, 2), (1_000_000, 4), (12_345_677, 7), (3, 3)):
        cap = oracle_mod.capacity(n, k)
        assert k * cap * 0.6 >= 1.15 * n


def test_budget_rule(oracle_mod):
    lib = oracle_mod._load()
    lib.oracle_budget.restype = ctypes.c_uint64
    lib.oracle_budget.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                  ctypes.c_uint64]
    # uniform primary counts -> theta0 x capacity (rounded down)
    assert lib.oracle_budget(100, 400, 4, 400_000, 1001) == 400
    # a cluster with 2x the mean primary share -> theta0 x capacity x 0.5
    assert lib.oracle_budget(200, 400, 4, 400_000, 1000) == 200
    # below the mean share -> min(1, .) caps at theta0 x capacity
    assert lib.oracle_budget(10, 400, 4, 400_000, 1000) == 400
    # no primaries yet
    assert lib.oracle_budget(0, 400, 4, 400_000, 1000) == 400
    # exact integer floor where fp64 would land at 0.999...: t*cap*min/(1e6*k*p) = 3*1/3
    assert lib.oracle_budget(3, 3, 1, 1_000_000, 1) == 1


def test_fig2_worked_example(oracle_mod):
    """PAPER P:300-302 preferences and P:364-366 outcome of Algorithm 1."""
    g = _golden("fig2_partition.json")
    C = np.array(g["centroids"], np.float32)
    X = np.array(g["points"], np.float32)
    d = oracle_mod.centroid_dist(X, C)
    assert np.allclose(d, np.array(g["expected_sq_dist"]), rtol=1e-6)
    for v, pref in enumerate(g["expected_preferences"]):
        assert np.argsort(d[v], kind="stable").tolist() == pref
    p = g["params"]
    r = oracle_mod.partition(X, C, omega=p["omega"], eps=p["eps"], theta0_ppm=p["theta0_ppm"],
                             alpha=p["alpha"], capacity=p["capacity"], block_size=p["block_size"])
    home = [[c for c in row if c != SENT] for row in r["home"].tolist()]
    exp = [[c for c in row if c is not None] for row in g["expected_home"]]
    assert home == exp
    assert np.allclose(r["radius"], g["expected_radius"], rtol=1e-6)
    for s, ids in enumerate(g["expected_idmaps"]):
        assert oracle_mod.idmap(r["home"], s).tolist() == ids


def test_fig2_fairness_v3_keeps_nearest(oracle_mod):
    """replicate-first order lets v1/v2 saturate c3 (cap 2) so v3 loses its
    nearest cluster; blockwise primaries-first keeps v3 on c3."""
    g = _golden("fig2_partition.json")
    C = np.array(g["centroids"], np.float32)
    X = np.array(g["points"][:3], np.float32)
    r = oracle_mod.partition(X, C, omega=2, eps=1000.0, theta0_ppm=999_999, alpha=1000.0, capacity=2)
    assert r["home"][2, 0] == 2          # v3's primary is c3 even with selectivity off
    assert (r["sizes"] <= 2).all()


def _rand_mixture(n, d, k, seed):
    rng = np.random.default_rng(seed)
    cen = rng.normal(size=(k, d)) * 4
    lab = rng.integers(0, k, n)
    return (cen[lab] + rng.normal(size=(n, d))).astype(np.float32)


@pytest.mark.parametrize("eps", [1.0, 0.9])
def test_eps_le_1_no_replicas(oracle_mod, eps):
    # SPEC S:210/S:236/S:255: d' >= d for the nearest primary, so eps <= 1 places no replica
    X = _rand_mixture(3000, 16, 8, 2)
    C = X[:8].copy()
    r = oracle_mod.partition(X, C, omega=3, eps=eps, block_size=512, capacity=3000)
    assert (r["home"][:, 1:] == SENT).all()
    # with ample capacity primaries equal brute-force nearest-centroid labels
    d = oracle_mod.centroid_dist(X, C)
    assert np.array_equal(r["home"][:, 0], np.argmin(d, axis=1))


def test_omega_1_no_replicas(oracle_mod):
    X = _rand_mixture(2000, 8, 4, 3)
    r = oracle_mod.partition(X, X[:4].copy(), omega=1, eps=3.0, block_size=256)
    assert r["home"].shape[1] == 1 and r["repl"].sum() == 0


@pytest.mark.parametrize("block", [65536, 700, 97])
def test_partition_invariants_and_audit(oracle_mod, block):
    X = _rand_mixture(4000, 12, 6, 4)
    C = X[::700][:6].copy()
    eps, alpha = 1.3, 1.0
    r = oracle_mod.partition(X, C, omega=3, eps=eps, alpha=alpha, block_size=block)
    home = r["home"]
    n, omega = home.shape
    cap = oracle_mod.capacity(n, 6)
    # coverage and omega bound, distinct homes
    assert (home[:, 0] != SENT).all()
    for row in home.tolist():
        real = [c for c in row if c != SENT]
        assert len(real) == len(set(real)) and 1 <= len(real) <= omega
        assert row[len(real):] == [SENT] * (omega - len(real))   # padding only at the tail
    sizes = np.array([(home == c).sum() for c in range(6)])
    assert np.array_equal(sizes, r["sizes"].astype(np.int64))
    assert (sizes <= cap).all()
    assert sizes.sum() == n + r["repl"].sum()
    # pruning soundness: every replica passes the distance constraint, and the
    # radius constraint with the largest tau (1+alpha) and the final radius (radius only grows)
    d = oracle_mod.centroid_dist(X, C)
    for v in range(n):
        p = home[v, 0]
        for c in home[v, 1:]:
            if c == SENT:
                continue
            assert d[v, c] < np.float32(eps) * d[v, p]
            assert d[v, c] < np.float32(eps) * np.float32(1 + alpha) * r["radius"][c]
    # replicated proportion is non-decreasing in eps — spot check
    r2 = oracle_mod.partition(X, C, omega=3, eps=1.6, alpha=alpha, block_size=block)
    assert r2["repl"].sum() >= r["repl"].sum()


def test_capacity_error(oracle_mod):
    X = _rand_mixture(100, 4, 2, 5)
    with pytest.raises(RuntimeError):
        oracle_mod.partition(X, X[:2].copy(), capacity=10)


# ---------------------------------------------------------------- P4 ----
def test_knn_line_by_hand(oracle_mod):
    # 1-D points 0,1,3,6,10 -> hand-computed nearest lists by (d^2, id)
    X = np.array([[0], [1], [3], [6], [10]], np.float32)
    ids, d = oracle_mod.knn(X, 3)
    assert ids.tolist() == [[1, 2, 3], [0, 2, 3], [1, 0, 3], [2, 4, 1], [3, 2, 1]]
    assert d.tolist() == [[1, 9, 36], [1, 4, 25], [4, 9, 9], [9, 16, 25], [16, 49, 81]]


def test_knn_tie_breaks_by_id(oracle_mod):
    X = np.array([[0], [1], [-1], [2], [-2]], np.uint8 if False else np.float32)
    ids, d = oracle_mod.knn(X, 4)
    assert ids[0].tolist() == [1, 2, 3, 4]          # equal distances -> lower id first
    assert d[0].tolist() == [1, 1, 4, 4]


def test_knn_m_equals_L_plus_1_and_padding(oracle_mod):
    rng = np.random.default_rng(7)
    X = rng.integers(0, 256, (9, 5)).astype(np.uint8)
    ids, _ = oracle_mod.knn(X, 8)                  # m = L+1 -> all other nodes
    for i in range(9):
        assert sorted(ids[i].tolist()) == [j for j in range(9) if j != i]
    ids, d = oracle_mod.knn(X, 10)                 # m - 1 < L -> sentinel / +inf padding
    assert (ids[:, 8:] == SENT).all() and np.isinf(d[:, 8:]).all()


def test_knn_inner_product_by_hand(oracle_mod):
    X = np.array([[1, 0], [0, 1], [2, 2], [3, 0]], np.float32)
    ids, d = oracle_mod.knn(X, 2, metric=1)        # dist = -<x, y>
    assert ids[0].tolist() == [3, 2] and d[0].tolist() == [-3, -2]


def test_knn_u8_exact_integer(oracle_mod):
    X = np.array([[255] * 4, [0] * 4, [255, 255, 255, 254]], np.uint8)
    ids, d = oracle_mod.knn(X, 2)
    assert d[1].tolist() == [255 * 255 * 3 + 254 * 254, 4 * 255 * 255]
    assert ids[0].tolist() == [2, 1]


# ---------------------------------------------------------------- P5/P6 ----
def test_prune_reverse_worked_example(oracle_mod):
    g = _golden("prune_reverse_example.json")
    X = np.array(g["points"], np.float32)
    ids, d = oracle_mod.knn(X, g["L"])
    assert ids.tolist() == g["expected_knn"]
    assert d[0].tolist() == g["expected_knn_sqdist_row0"]
    p, pd = oracle_mod.prune(ids, d, g["R"], rule=0)
    assert p.tolist() == g["expected_pruned_ruleP"]
    p1, _ = oracle_mod.prune(ids, d, g["R"], rule=1)
    assert p1[1].tolist() == g["expected_pruned_relaxed_node1"]
    f, fd = oracle_mod.reverse(p, pd, protected=1)
    assert f.tolist() == g["expected_final_h1"]
    rev, _, rc = oracle_mod.reverse_lists(p, pd)
    assert [rev[y, :rc[y]].tolist() for y in range(len(rc))] == g["expected_reverse_lists"]
    # carried distance of a reverse edge y->x is the distance of x->y
    assert fd[1, 1] == pd[5, 1] and fd[2, 1] == pd[0, 1]


def test_reverse_capped_order_is_rank_then_source(oracle_mod):
    """R11's (k, x) order decides which sources survive the cap when in-degree > R
    (tests/golden/reverse_order_example.json, hand-derived)."""
    g = _golden("reverse_order_example.json")
    p = np.array(g["pruned"], np.uint32)
    pd = np.array(g["pruned_d"], np.float32)
    rev, rd, rc = oracle_mod.reverse_lists(p, pd)
    assert [rev[y, :rc[y]].tolist() for y in range(4)] == g["expected_reverse_lists"]
    assert [rd[y, :rc[y]].tolist() for y in range(4)] == g["expected_reverse_lists_d"]
    f, fd = oracle_mod.reverse(p, pd, protected=g["h"])
    assert f.tolist() == g["expected_final"]
    assert f[3].tolist() != g["expected_final_if_xk_order_node3"]
    assert fd[3].tolist() == [4.0, 3.0]     # protected edge keeps d(3 -> 1), reverse edge carries d(2 -> 3)


def test_prune_rank_lookup_matches_brute_force(oracle_mod):
    """P5 by brute force over (r_ad, r_db, r_ab) in Python on a small random graph."""
    rng = np.random.default_rng(5)
    X = rng.normal(size=(60, 3)).astype(np.float32)
    L, R = 8, 5
    ids, d = oracle_mod.knn(X, L)
    for rule in (0, 1):
        p, _ = oracle_mod.prune(ids, d, R, rule=rule)
        for a in range(60):
            cnt = [0] * L
            for r_ad in range(L):
                dl = ids[a, r_ad]
                for r_db in range(L):
                    b = ids[dl, r_db]
                    if b == a:
                        continue
                    for r_ab in range(L):
                        if ids[a, r_ab] == b:
                            mx = max(r_ad, r_db) if rule == 0 else r_ad
                            cnt[r_ab] += mx < r_ab
            order = sorted(range(L), key=lambda r: (cnt[r], r))[:R]
            assert p[a].tolist() == [int(ids[a, r]) for r in order]


def test_prune_invariants(oracle_mod):
    rng = np.random.default_rng(11)
    X = rng.normal(size=(300, 6)).astype(np.float32)
    L, R = 16, 8
    ids, d = oracle_mod.knn(X, L)
    p, pd = oracle_mod.prune(ids, d, R)
    for a in range(300):
        assert set(p[a].tolist()) <= set(ids[a].tolist())       # output subset of N[a]
        assert p[a, 0] == ids[a, 0]                              # rank 0 always first
        assert len(set(p[a].tolist())) == R
    full, _ = oracle_mod.prune(ids, d, L)                        # L = R -> a permutation
    assert all(sorted(full[a]) == sorted(ids[a]) for a in range(300))


def test_reverse_invariants(oracle_mod):
    rng = np.random.default_rng(12)
    X = rng.normal(size=(400, 5)).astype(np.float32)
    ids, d = oracle_mod.knn(X, 12)
    p, pd = oracle_mod.prune(ids, d, 8)
    f, fd = oracle_mod.reverse(p, pd)
    for y in range(400):
        row = f[y].tolist()
        assert len(set(row)) == 8 and y not in row               # fixed degree, no dup/self
        assert row[:4] == p[y, :4].tolist()                      # protected prefix kept
        assert set(row) <= set(p[y].tolist()) | {x for x in range(400) if y in p[x].tolist()}
    # no reverse edges (all rows point to a single sink-free cycle) -> out = pruned
    cyc = np.array([[(i + 1) % 5, (i + 2) % 5] for i in range(5)], np.uint32)
    cyc_d = np.ones((5, 2), np.float32)
    out, _ = oracle_mod.reverse(cyc, cyc_d, protected=2)
    assert np.array_equal(out, cyc)


# ---------------------------------------------------------------- P7 ----
def test_merge_single_shard_identity(oracle_mod):
    # one shard with identity idmap -> merged = shard graph
    rng = np.random.default_rng(13)
    X = rng.normal(size=(200, 4)).astype(np.float32)
    ids, d = oracle_mod.knn(X, 8)
    home = np.zeros((200, 1), np.uint32)
    m, md = oracle_mod.merge(home, [np.arange(200, dtype=np.uint32)], [ids], [d])
    assert np.array_equal(m, ids) and np.array_equal(md, d)


def test_merge_union_example(oracle_mod):
    # rows {a,b} and {b,c} -> {a,b,c}; here R=3 so the union fits
    home = np.array([[0, 1], [0, SENT], [0, 1], [1, SENT]], np.uint32)
    idm = [np.array([0, 1, 2], np.uint32), np.array([0, 2, 3], np.uint32)]
    g0 = np.array([[1, 2, SENT], [0, 2, SENT], [0, 1, SENT]], np.uint32)
    g0d = np.array([[1, 2, np.inf], [1, 3, np.inf], [2, 3, np.inf]], np.float32)
    g1 = np.array([[1, 2, SENT], [0, 2, SENT], [0, 1, SENT]], np.uint32)   # locals of shard 1
    g1d = np.array([[4, 5, np.inf], [4, 6, np.inf], [5, 6, np.inf]], np.float32)
    m, md = oracle_mod.merge(home, idm, [g0, g1], [g0d, g1d])
    assert m[0].tolist() == [1, 2, 3] and md[0].tolist() == [1, 2, 5]      # {1,2} u {2,3}
    assert m[1].tolist() == [0, 2, SENT]                                     # single home as is
    assert m[3].tolist() == [0, 2, SENT]                                     # shard-1 locals mapped


def test_merge_order_independent_and_truncation(oracle_mod):
    # SPEC S:414 order independence, S:415 truncation optimality
    rng = np.random.default_rng(14)
    X = rng.normal(size=(300, 4)).astype(np.float32)
    C = X[:3].copy()
    r = oracle_mod.partition(X, C, omega=2, eps=2.0)
    R = 6
    idm, gs, gds = [], [], []
    for s in range(3):
        im = oracle_mod.idmap(r["home"], s)
        ids, d = oracle_mod.knn(X, R, ida=im)
        idm.append(im), gs.append(ids), gds.append(d)
    m, md = oracle_mod.merge(r["home"], idm, gs, gds)
    for g in range(300):
        homes = [c for c in r["home"][g] if c != SENT]
        if len(homes) < 2:
            continue
        cand = {}
        for s in homes:
            l = int(np.searchsorted(idm[s], g))
            for j in range(R):
                gid = int(idm[s][gs[s][l, j]])
                cand[gid] = min(cand.get(gid, np.inf), float(gds[s][l, j]))
        kept = m[g].tolist()
        assert set(kept) <= set(cand)
        worst_kept = max(cand[k] for k in kept)
        assert all(v >= worst_kept for k, v in cand.items() if k not in kept)
    # S:414 order independence: the union of a multi-home row does not depend on the order of
    # the entries within each home's row, nor on the order of the homes in home[g]
    perm_gs, perm_gds = [], []
    for s in range(3):
        pr = np.argsort(rng.random(gs[s].shape), axis=1)
        perm_gs.append(np.take_along_axis(gs[s], pr, 1))
        perm_gds.append(np.take_along_axis(gds[s], pr, 1))
    home_sw = r["home"].copy()
    multi = (home_sw != SENT).sum(1) > 1
    home_sw[multi] = home_sw[multi][:, ::-1]
    assert multi.sum() > 20
    m2, md2 = oracle_mod.merge(home_sw, idm, perm_gs, perm_gds)
    assert np.array_equal(m[multi], m2[multi]) and np.array_equal(md[multi], md2[multi])
    # single-home rows are taken as is (in their shard's row order)
    single = ~multi
    assert not np.array_equal(m[single], m2[single])
    for g in np.nonzero(single)[0][:50]:
        s = int(r["home"][g, 0])
        l = int(np.searchsorted(idm[s], g))
        assert m2[g].tolist() == idm[s][perm_gs[s][l]].tolist()


def test_entry_points(oracle_mod):
    home = np.array([[0, SENT], [1, 0], [0, SENT], [1, SENT]], np.uint32)
    pd = np.array([3.0, 1.0, 2.0, 5.0], np.float32)
    g, per = oracle_mod.entry_points(home, pd, [3, 2])
    assert per.tolist() == [2, 1] and g == 2       # shard 0 is the larger: its entry


# ---------------------------------------------------------------- P8 ----
def test_search_full_beam_is_exact(oracle_mod):
    # beam = n on a connected graph -> exact top-k (the P4 definition)
    rng = np.random.default_rng(15)
    X = rng.normal(size=(150, 6)).astype(np.float32)
    ids, _ = oracle_mod.knn(X, 10)
    ring = np.array([[(i + 1) % 150] for i in range(150)], np.uint32)
    graph = np.concatenate([ids, ring], axis=1)               # ring makes it connected
    Q = rng.normal(size=(20, 6)).astype(np.float32)
    res, dd, nd = oracle_mod.search(X, graph, 0, Q, topk=10, beam=150)
    gt, _ = oracle_mod.knn(Q, 10, xb=X, self_exclude=False)
    assert np.array_equal(res, gt)
    assert (nd == 150).all()                                  # every node evaluated once
    assert oracle_mod.recall(gt, gt) == 1.0


def test_search_shards_disconnected_full_beam_is_exact(oracle_mod):
    # Split-only graph: two disjoint shards, each a ring-connected kNN graph of its
    # own members.  One beam from a single entry cannot leave its shard; one full beam per
    # shard entry + the merge of the results must give the exact top-k over all points.
    rng = np.random.default_rng(18)
    X = rng.normal(size=(160, 5)).astype(np.float32)
    parts = [np.arange(0, 160, 2), np.arange(1, 160, 2)]
    graph = np.full((160, 9), 0xFFFFFFFF, np.uint32)
    for ids_s in parts:
        loc, _ = oracle_mod.knn(X[ids_s], 8)
        graph[ids_s, :8] = ids_s[loc]
        graph[ids_s, 8] = np.roll(ids_s, -1)
    Q = rng.normal(size=(15, 5)).astype(np.float32)
    gt, _ = oracle_mod.knn(Q, 10, xb=X, self_exclude=False)
    res = oracle_mod.search_shards(X, graph, [0, 1], Q, topk=10, beam=80)
    assert np.array_equal(res, gt)
    one, _, nd = oracle_mod.search(X, graph, 0, Q, topk=10, beam=80)
    assert (one % 2 == 0).all() and (nd == 80).all()          # a single beam stays in shard 0


def test_search_query_is_data_point(oracle_mod):
    rng = np.random.default_rng(16)
    X = rng.normal(size=(100, 3)).astype(np.float32)
    ids, _ = oracle_mod.knn(X, 8)
    res, dd, _ = oracle_mod.search(X, ids, 0, X[[5, 17]], topk=3, beam=32)
    assert res[0, 0] == 5 and res[1, 0] == 17 and dd[0, 0] == 0


# ---------------------------------------------------------------- P0 ----
def test_kmeans_distortion_by_hand(oracle_mod):
    """The distortion that judges the GPU k-means (R0): sum over the sample of the squared
    distance to the nearest centroid.  Hand values: points 0, 2, 10, 13 on a line with
    centroids 1 and 10 give 1 + 1 + 0 + 9 = 11; the sample floor(i n / S) with S = min(n, spc k)
    = 2 (spc = 1, k = 2) is rows 0 and 2: 1 + 0 = 1."""
    X = np.array([[0, 0], [2, 0], [10, 0], [13, 0]], np.float32)
    C = np.array([[1, 0], [10, 0]], np.float32)
    assert oracle_mod.kmeans_distortion(X, C, spc=256) == 11.0
    assert oracle_mod.kmeans_distortion(X, C, spc=1) == 1.0
    assert oracle_mod.kmeans_distortion(X, C[::-1].copy(), spc=256) == 11.0


def test_kmeans_k1_is_mean(oracle_mod):
    rng = np.random.default_rng(17)
    X = rng.normal(size=(500, 7)).astype(np.float32)
    C, _ = oracle_mod.kmeans(X, 1, spc=1000)
    assert np.allclose(C[0], X.astype(np.float64).mean(0), atol=1e-6)


def test_kmeans_distinct_points_zero_distortion(oracle_mod):
    X = np.repeat(np.array([[0, 0], [5, 5], [10, 0]], np.float32), 20, axis=0)
    C, dist = oracle_mod.kmeans(X, 3, spc=20)
    assert dist == 0.0
    assert sorted(map(tuple, C.tolist())) == [(0, 0), (5, 5), (10, 0)]


def test_kmeans_monotone_and_deterministic(oracle_mod):
    X = _rand_mixture(2000, 8, 6, 18)
    ds = [oracle_mod.kmeans(X, 6, seed=3, max_iter=i)[1] for i in range(6)]
    assert all(b <= a * (1 + 1e-12) for a, b in zip(ds, ds[1:]))
    C1, _ = oracle_mod.kmeans(X, 6, seed=3)
    C2, _ = oracle_mod.kmeans(X, 6, seed=3)
    assert np.array_equal(C1, C2)
