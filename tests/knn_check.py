"""The kNN acceptance rule of DESIGN.md (north_star: distances within 1e-3 relative, fp32
accumulated; ids identical except among ties within that tolerance).  Per row i, with
tol(x) = 1e-3*|x| + 1e-6*(|x_i|^2 + max_j |x_j|^2):
  1. |G.d[p] - O.d[p]| <= tol(O.d[p]) for every position p;
  2. every oracle id with O.d < tau_L - tol(tau_L) appears in G (tau_L = O.d[L-1]);
  3. every GPU id not in the oracle list has exact distance <= tau_L + tol(tau_L);
  4. G has no duplicates, no self, and no sentinel unless fewer than L candidates exist.
Exact pair distances for rule 3 are recomputed in float64 (the P4 definition).
"""
import numpy as np

SENT = 0xFFFFFFFF


def exact_pair(xa, xb, i, j, metric=0):
    a = xa[i].astype(np.float64)
    b = xb[j].astype(np.float64)
    return float(((a - b) ** 2).sum()) if metric == 0 else float(-(a * b).sum())


def check_knn(G_ids, G_d, O_ids, O_d, xa, xb=None, self_exclude=True, metric=0, rel=1e-3, abs_scale=1e-6):
    """Returns (n_rows_failed, first_failure_message)."""
    xb = xa if xb is None else xb
    G_ids = np.asarray(G_ids).astype(np.uint32)
    O_ids = np.asarray(O_ids).astype(np.uint32)
    G_d = np.asarray(G_d, np.float64)
    O_d = np.asarray(O_d, np.float64)
    ma, L = O_ids.shape
    na = (xa.astype(np.float64) ** 2).sum(1)
    maxb = float((xb.astype(np.float64) ** 2).sum(1).max())
    fails, first = 0, None
    for i in range(ma):
        floor = abs_scale * (na[i] + maxb) if metric == 0 else abs_scale * (na[i] + maxb)
        tol = lambda v: rel * abs(v) + floor  # noqa: E731
        msg = None
        g, o = G_ids[i], O_ids[i]
        real_o = o != SENT
        if not np.array_equal(g == SENT, ~real_o):
            msg = f"row {i}: sentinel pattern differs"
        else:
            diff = np.abs(G_d[i][real_o] - O_d[i][real_o])
            bad = diff > np.array([tol(v) for v in O_d[i][real_o]])
            if bad.any():
                p = int(np.nonzero(bad)[0][0])
                msg = f"row {i} pos {p}: gpu {G_d[i][p]} oracle {O_d[i][p]}"
        if msg is None:
            gs = set(g[g != SENT].tolist())
            if len(gs) != int((g != SENT).sum()):
                msg = f"row {i}: duplicate ids"
            elif self_exclude and i in gs:
                msg = f"row {i}: self loop"
        if msg is None and real_o.any():
            tau = O_d[i][real_o][-1]
            os_ = set(o[real_o].tolist())
            must = set(o[(O_d[i] < tau - tol(tau)) & real_o].tolist())
            if not must <= gs:
                msg = f"row {i}: missing clear neighbours {sorted(must - gs)[:5]}"
            else:
                for j in gs - os_:
                    dj = exact_pair(xa, xb, i, j, metric)
                    if dj > tau + tol(tau):
                        msg = f"row {i}: extra id {j} at {dj} > tau {tau}"
                        break
        if msg is not None:
            fails += 1
            first = first or msg
    return fails, first
