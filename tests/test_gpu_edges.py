"""Error paths and degenerate cases on the GPU, each against the oracle:
SG_ERR_CAPACITY raised by GPU and oracle alike, SG_ERR_TOO_SMALL, prune
and reverse of sentinel-padded kNN rows (m - 1 < L), k = 1, an empty shard, and byte-identical
reruns (determinism)."""
import numpy as np
import pytest
import torch

from paper_2605_10135_b200 import datagen

pytestmark = pytest.mark.gpu
SENT = 0xFFFFFFFF


@pytest.fixture(scope="module")
def api():
    from paper_2605_10135_b200 import api as a
    a.load()
    return a


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def test_capacity_error_gpu_and_oracle(api, oracle_mod):
    """Capacity = n/k with aggressive replication (theta0 = 0.9, eps = 3): replicas of the first
    blocks fill the clusters and a later primary finds every cluster full."""
    x = datagen.sift_like(4000, 32, seed=81)
    C = x[::1000][:4].clone()
    kw = dict(omega=2, theta0_ppm=900_000, capacity=1000, block_size=256)
    with pytest.raises(RuntimeError, match="CAPACITY"):
        oracle_mod.partition(x.numpy(), C.numpy(), eps=3.0, **kw)
    with pytest.raises(api.ScaleGannError) as ei:
        api.scalegann_partition(x.cuda(), C.cuda(), epsilon=3.0, **kw)
    assert ei.value.status == 4


def test_shard_too_small(api):
    x = datagen.sift_like(100, 32, seed=82).cuda()
    idm = torch.tensor([5], dtype=torch.int32, device="cuda")
    with pytest.raises(api.ScaleGannError) as ei:
        api.scalegann_build_shard(x, idm, 16, 8)
    assert ei.value.status == 6


@pytest.mark.parametrize("m,L,R", [(20, 32, 16), (9, 16, 16), (2, 8, 4)])
def test_prune_reverse_sentinel_padded(api, oracle_mod, m, L, R):
    """Shards smaller than L + 1: kNN rows padded with (SENT, +inf); prune and reverse keep
    the padding rules of P5 (sentinel ranks last) and P6 bit for bit."""
    x = datagen.sift_like(m, 32, seed=83 + m)
    ki, kd = api.scalegann_knn(x.cuda(), L)
    oi, od = oracle_mod.knn(x.numpy(), L)
    assert np.array_equal(u32(ki), oi) and np.array_equal(kd.cpu().numpy(), od)
    assert (oi == SENT).any()
    g, gd = api.scalegann_optimize_from_knn(ki, kd, R)
    pr, prd = oracle_mod.prune(oi, od, R)
    f, fd = oracle_mod.reverse(pr, prd)
    assert np.array_equal(u32(g), f) and np.array_equal(gd.cpu().numpy(), fd)


def _oracle_graph(oracle_mod, x, C, cfg, capacity=0):
    r = oracle_mod.partition(x, C, omega=cfg.omega, eps=cfg.epsilon, block_size=cfg.block_size, capacity=capacity)
    idm, gs, gds = [], [], []
    for s in range(cfg.k):
        im = oracle_mod.idmap(r["home"], s)
        if len(im) == 0:
            idm.append(im), gs.append(np.zeros((0, cfg.R), np.uint32)), gds.append(np.zeros((0, cfg.R), np.float32))
            continue
        ids, dd = oracle_mod.knn(x, cfg.L, ida=im)
        pr, prd = oracle_mod.prune(ids, dd, cfg.R)
        f, fd = oracle_mod.reverse(pr, prd)
        idm.append(im), gs.append(f), gds.append(fd)
    return r, oracle_mod.merge(r["home"], idm, gs, gds)


def test_single_shard_k1(api, oracle_mod):
    from paper_2605_10135_b200.pipeline import BuildConfig, build_index
    x = datagen.sift_like(3000, 64, seed=84)
    cfg = BuildConfig(k=1, omega=1, L=32, R=16, block_size=1024)
    idx = build_index(x.cuda(), cfg)
    r, (om, omd) = _oracle_graph(oracle_mod, x.numpy(), idx.centroids.cpu().numpy(), cfg)
    assert np.array_equal(u32(idx.home), r["home"])
    assert np.array_equal(u32(idx.merged), om) and np.array_equal(idx.merged_d.cpu().numpy(), omd)


def test_empty_shard(api, oracle_mod):
    """A centroid far from every vector: its shard stays empty (no build, entry SENTINEL) and the
    merged graph still equals the oracle's."""
    from paper_2605_10135_b200.pipeline import BuildConfig, lpt_owner
    x = datagen.sift_like(4000, 64, seed=85)
    C = torch.cat([x[::2000][:2], torch.full((1, 64), 1e6)]).contiguous()
    cfg = BuildConfig(k=3, omega=2, L=32, R=16, block_size=1024)
    # capacity 4000: the two near clusters never fill, so no primary spills to the far one
    home, pd, counts = api.scalegann_partition(x.cuda(), C.cuda(), omega=2, epsilon=cfg.epsilon,
                                               block_size=cfg.block_size, capacity=4000)
    assert counts["sizes"][2] == 0
    idm, gs, gds = [], [], []
    for s in range(3):
        if counts["sizes"][s] == 0:
            idm.append(None), gs.append(None), gds.append(None)
            continue
        idm.append(api.scalegann_shard_idmap(home, s, m=counts["sizes"][s]))
        g, gd = api.scalegann_build_shard(x.cuda(), idm[-1], cfg.L, cfg.R)
        gs.append(g), gds.append(gd)
    merged, merged_d = api.scalegann_merge(home, idm, gs, gds)
    r, (om, omd) = _oracle_graph(oracle_mod, x.numpy(), C.numpy(), cfg, capacity=4000)
    assert np.array_equal(u32(home), r["home"])
    assert np.array_equal(u32(merged), om) and np.array_equal(merged_d.cpu().numpy(), omd)
    g, per = api.scalegann_entry_points(home, pd, counts["sizes"])
    assert per[2] == SENT and g != SENT


@pytest.mark.parametrize("kind", ["sift", "deep"])
def test_rerun_is_byte_identical(api, kind):
    """Two builds of the same data give the same bytes (atomics inside the kernels never leak
    into the results: every selection ends in a (dist, id) sort)."""
    from paper_2605_10135_b200.pipeline import BuildConfig, build_index
    x = datagen._make(kind, 20_000, 96, 86, "cuda")
    cfg = BuildConfig(k=3, L=64, R=32)
    a = build_index(x, cfg)
    b = build_index(x, cfg)
    assert torch.equal(a.home, b.home) and torch.equal(a.merged, b.merged) and torch.equal(a.merged_d, b.merged_d)


def test_build_index_host_equals_pipeline(api):
    """The one-call host-buffer entry point (bench's e2e path) builds the pipeline's graph."""
    from paper_2605_10135_b200.pipeline import BuildConfig, build_index
    x = datagen.sift_like(12_000, 64, seed=87)
    cfg = BuildConfig(k=3, L=64, R=32)
    ref = build_index(x.cuda(), cfg)
    out = torch.empty(12_000 * 32, dtype=torch.int32).pin_memory()
    outd = torch.empty(12_000 * 32, dtype=torch.float32).pin_memory()
    no, entry = api.scalegann_build_index_host(x.pin_memory(), out, k=3, L_=64, R=32, merged_d_host=outd)
    assert no == 12_000 and entry == ref.entry
    assert torch.equal(out.view(-1, 32), ref.merged.cpu()) and torch.equal(outd.view(-1, 32), ref.merged_d.cpu())
