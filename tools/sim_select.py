"""CPU simulation of the transposed kernel's per-row selection dynamics (policy exploration only:
no part of the method's arithmetic).  One row, m columns in random order, 128-column tiles, NS=4
streams of 32 columns each; counts events (a stream's 32-column chunk with >= 1 candidate),
insertions, compactions and whether the final exactness check passes."""
import argparse
import numpy as np


def sim_row(rng, m, L, CS, alpha, beta, eager=0, refresh=False):
    keys = rng.random(m)
    ntile = m // 128
    thr = np.inf
    bufs = [[] for _ in range(4)]
    ev = ins = comp = 0
    for t in range(ntile):
        f = (t + 1) / ntile
        for q in range(4):
            blk = keys[t * 128 + 32 * q: t * 128 + 32 * q + 32]
            sel = blk[blk <= thr]
            if len(sel):
                ev += 1
                ins += len(sel)
                bufs[q].extend(sel.tolist())
            lim = CS - 32 if not eager else None
            want = min(L, int(alpha * L * f / 4) + beta)
            kmax = want + (CS - 32 - want) // 8
            trigger = len(bufs[q]) > CS - 32 or (eager and len(bufs[q]) >= want + eager)
            if trigger:
                comp += 1
                b = sorted(x for x in bufs[q] if x <= thr)
                if refresh:   # row-level: want-th over all streams' entries (x4 rank)
                    allk = sorted(x for s in range(4) for x in bufs[s] if x <= thr)
                    w4 = min(L, int(alpha * L * f) + 4 * beta)
                    if len(allk) > w4:
                        thr = min(thr, allk[w4 - 1])
                    b = [x for x in b if x <= thr]
                elif len(b) > kmax and len(b) >= want:
                    thr = min(thr, b[want - 1])
                    b = [x for x in b if x <= thr]
                bufs[q] = b
    allk = sorted(x for s in range(4) for x in bufs[s] if x <= thr)
    ok = len(allk) >= L
    return ev, ins, comp, ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=400_000)
    ap.add_argument("--L", type=int, default=128)
    ap.add_argument("--rows", type=int, default=20)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    for CS, alpha, beta, eager, refresh in [(128, 1.5, 8, 0, False), (64, 1.5, 8, 0, False), (128, 1.5, 8, 16, False),
                                            (128, 1.5, 4, 16, False), (128, 1.5, 8, 0, True), (128, 1.5, 4, 16, True),
                                            (128, 1.5, 2, 8, True), (256, 1.5, 8, 0, True)]:
        r = np.array([sim_row(rng, a.m, a.L, CS, alpha, beta, eager, refresh) for _ in range(a.rows)], dtype=float)
        print(f"CS={CS} a={alpha} b={beta} eager={eager} refresh={refresh}: events {r[:,0].mean():.0f} "
              f"ins {r[:,1].mean():.0f} comp {r[:,2].mean():.1f} fail {1 - r[:,3].mean():.2f}")


if __name__ == "__main__":
    main()
