"""CPU model of the device launch pipeline (for host-logic tests without a GPU).

Launch j maps A_{j-1} -> A_j and yields, exactly as K1 + fold do on the device
(SURVEY.md Appendix B): step_j, max|A_j|, nonfinite(A_j), the row residuals of
A_{j-1}; the cycle kernel then yields the "not within" flags of A_j against the
window.  The statistics are consumed by the SAME decision function the device
runs (dpt_sm_decide_host in libdpt_b200.so).  With rows=(r0, r1) only that row
shard is computed and the caller combines shards (max) -- the multi-GPU path.
"""
import ctypes

import numpy as np

import paper_2002_12872_b200._native as N

NSTATS = 20


class SmState:
    def __init__(self, opts, win, trace=False):
        L = N.lib()
        self.buf = ctypes.create_string_buffer(int(L.dpt_sm_state_bytes()) + 64)
        self.obuf = ctypes.create_string_buffer(256)
        o = N.dpt_options(opts.get("tol", 1e-12), opts.get("residual_tol", 1e-10), int(opts.get("max_iter", 10000)),
                          opts.get("divergence_threshold", 1e8), int(opts.get("cycle_window", 16)),
                          opts.get("degeneracy_tol", 1e-12))
        L.dpt_sm_init(self.buf, self.obuf, ctypes.byref(o), int(win), 1 if trace else 0)
        self.trace = np.zeros(3 * (int(opts.get("max_iter", 10000)) + 2))

    def decide(self, stats, j):
        s = np.ascontiguousarray(stats, dtype=np.float64)
        N.lib().dpt_sm_decide_host(self.buf, self.obuf, s.ctypes.data, int(j), 1, 1, self.trace.ctypes.data)

    def query(self):
        v = [ctypes.c_int() for _ in range(6)]
        step = ctypes.c_double()
        N.lib().dpt_sm_query(self.buf, *[ctypes.byref(x) for x in v], ctypes.byref(step))
        done, status, iters, final_iter, readoffs, cycle_pending = (x.value for x in v)
        return dict(done=done, status=status, iterations=iters, final_iter=final_iter, readoffs=readoffs,
                    cycle_pending=cycle_pending, step_norm=step.value)


def dense_of(p):
    return p.delta.todense() if hasattr(p.delta, "rowptr") else np.asarray(p.delta)


def launch_rows(p, a_prev_rows, r0, lam_k, D):
    """Rows [r0, r0+len) of A_j = F(A_{j-1}) in the reference's operation order
    (matmul P = A Delta^T, then the map), plus the shard's stats pieces."""
    d, lam = np.asarray(p.d), p.lam
    rows, n = a_prev_rows.shape
    P = a_prev_rows @ D.T
    gi = np.arange(r0, r0 + rows)
    pii = P[np.arange(rows), gi]
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        th = 1.0 / (d[gi][:, None] - d[None, :])
        an = (lam_k * th) * (P - pii[:, None] * a_prev_rows)
    an[np.arange(rows), gi] = 1.0
    eps = d[gi] + lam * pii
    with np.errstate(invalid="ignore", over="ignore"):
        r = (d[None, :] - eps[:, None]) * a_prev_rows + lam * P
    num = np.nanmax(np.abs(r), axis=1)
    den = np.nanmax(np.abs(a_prev_rows), axis=1)
    res = num / np.maximum(den, 1e-300)
    with np.errstate(invalid="ignore"):
        step = float(np.nanmax(np.abs(an - a_prev_rows))) if an.size else 0.0
        mx = float(np.nanmax(np.abs(an))) if an.size else 0.0
    nonfin = float(np.count_nonzero(~np.isfinite(an)))
    return an, dict(step=step, maxabs=mx, nonfin=nonfin, maxres=float(np.max(res)) if res.size else 0.0,
                    eps=eps, res=res)


def cycle_flags(a_j, window, tol):
    """flags[p] = 1 unless within_tol(A_j, window[p]) (dpt.cpp:60-79)."""
    f = np.ones(16)
    for q, past in enumerate(window):
        with np.errstate(invalid="ignore"):
            f[q] = 0.0 if not np.any(np.abs(a_j - past) >= tol) else 1.0
    return f


def simulate(p, opts, allreduce=None, shard=None):
    """Runs the launch pipeline.  shard=(r0, r1) computes only those rows and
    `allreduce(vec) -> vec` combines the statistics vector (max over ranks)."""
    n = len(p.d)
    D = dense_of(p)
    max_iter = int(opts.get("max_iter", 10000))
    tol = opts.get("tol", 1e-12)
    req = int(opts.get("cycle_window", 16))
    cap = 4.0e6 / max(float(n) * n, 1.0)
    win = req if req > 0 else 0
    if req > 0 and cap < win:
        win = int(cap)
    win = win if win >= 2 else 0
    r0, r1 = shard or (0, n)
    sm = SmState(opts, win)
    hist = {0: np.eye(n)[r0:r1]}
    a = hist[0]
    cyc = np.ones(16)
    reads = {}
    for j in range(1, max_iter + 2):
        an, st = launch_rows(p, a, r0, p.lam, D)
        reads[j - 1] = (st["eps"], st["res"])
        vec = np.zeros(NSTATS)
        vec[0], vec[1], vec[2], vec[3] = st["step"], st["maxabs"], st["nonfin"], st["maxres"]
        vec[4:20] = cyc
        if allreduce:
            vec = allreduce(vec)
        sm.decide(vec, j)
        hist[j] = an
        q = sm.query()
        if q["done"]:
            break
        cyc = np.ones(16)
        if q["cycle_pending"]:
            npast = min(j - 1, win - 1)
            cyc = cycle_flags(an, [hist[j - 2 - k] for k in range(npast)], tol)
        a = an
    q = sm.query()
    m = q["final_iter"]
    eps, res = reads.get(m, (np.full(r1 - r0, np.nan), np.full(r1 - r0, np.nan)))
    if not q["readoffs"]:
        eps, res = np.full(r1 - r0, np.nan), np.full(r1 - r0, np.nan)
    return q, hist[m], eps, res
