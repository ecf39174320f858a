"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

CPU restatement of the reference sampling strategies
(pkg/src/parastep/engines.py). A predictor is any callable
``pred(x, t, T) -> eps`` on float64 vectors.

Outputs are plain dicts/lists so tests can compare them with the GPU product
path without importing either side's classes:

    traj = {"t": [...], "x": [vec...], "eps": [vec...], "fresh": [...], "x0": vec}
"""

from __future__ import annotations

import numpy as np

from .core import P_INIT, P_STEP, Sched, ddpm_step, make_stream, normals


def x_init(seed: int, n: int) -> np.ndarray:
    """initial_state: stream (INIT<<32)|0 (engines.py:172-174)."""
    return normals(seed, make_stream(P_INIT, 0), n)


def z_step(seed: int, t: int, n: int) -> np.ndarray:
    """step_noise: stream (STEP<<32)|t (engines.py:177-179)."""
    return normals(seed, make_stream(P_STEP, t), n)


def _warm(T: int, warmup: int, t: int) -> bool:
    return (T - t) < warmup  # engines.py:192-193


def _new_traj():
    return {"t": [], "x": [], "eps": [], "fresh": [], "x0": None}


def _rec(tr, t, x, eps, fresh):
    tr["t"].append(t)
    tr["x"].append(x)
    tr["eps"].append(eps)
    tr["fresh"].append(bool(fresh))


def sequential(pred, sch: Sched, n: int, seed: int):
    """engines.py:196-205."""
    tr = _new_traj()
    x = x_init(seed, n)
    for t in range(sch.T, 0, -1):
        e = pred(x, t, sch.T)
        _rec(tr, t, x, e, True)
        x = ddpm_step(x, t, e, sch, z_step(seed, t, n))
    tr["x0"] = x
    return tr


def direct_reuse(pred, sch: Sched, n: int, seed: int, warmup: int, stride: int):
    """engines.py:208-229."""
    tr = _new_traj()
    x = x_init(seed, n)
    last = None
    k = 0
    for t in range(sch.T, 0, -1):
        if _warm(sch.T, warmup, t):
            fresh = True
        else:
            fresh = k % stride == 0
            k += 1
        if fresh:
            last = pred(x, t, sch.T)
        _rec(tr, t, x, last, fresh)
        x = ddpm_step(x, t, last, sch, z_step(seed, t, n))
    tr["x0"] = x
    return tr


def parastep_algorithm1(pred, sch: Sched, n: int, seed: int, warmup: int, p: int):
    """Algorithm 1 with p lockstep virtual ranks (engines.py:232-277).

    Returns (traj of rank 0, per-rank histories) where a history entry is
    (t, x_before, eps, source, x_after) and source is one of
    "local_fresh" / "remote_fresh" / "reuse".
    """
    tr = _new_traj()
    x0 = x_init(seed, n)
    xs = [x0] * p
    cache = [None] * p
    hist = [[] for _ in range(p)]
    rnd = 0
    for t in range(sch.T, 0, -1):
        z = z_step(seed, t, n)
        warm = _warm(sch.T, warmup, t)
        m = 0 if warm else rnd
        before = list(xs)
        e_m = pred(before[m], t, sch.T)
        for r in range(p):
            if warm or r == m:
                e, src = e_m, "local_fresh"
                cache[r] = e_m
            elif r == 0:
                e, src = e_m, "remote_fresh"
            else:
                e, src = cache[r], "reuse"
            xs[r] = ddpm_step(before[r], t, e, sch, z)
            hist[r].append([t, before[r], e, src, xs[r]])
        _rec(tr, t, before[0], e_m, warm or m == 0)
        if not warm:
            if rnd == p - 1:
                for r in range(1, p):
                    xs[r] = xs[0]
                    hist[r][-1][4] = xs[0]
            rnd = (rnd + 1) % p
    tr["x0"] = xs[0]
    return tr, hist


def plan_cycles(T: int, warmup: int, degree: int, lengths=None) -> list[list[int]]:
    """Post-warm-up steps chunked into cycles (engines.py:280-296)."""
    ts = list(range(T - warmup, 0, -1))
    if lengths is None:
        lengths, left = [], len(ts)
        while left > 0:
            lengths.append(min(degree, left))
            left -= lengths[-1]
    out, pos = [], 0
    for c in lengths:
        out.append(ts[pos:pos + c])
        pos += c
    return out


def cycles(pred, sch: Sched, n: int, seed: int, warmup: int, degree: int, lengths=None):
    """Cycle runner shared by batchstep / dynamic (engines.py:299-337)."""
    tr = _new_traj()
    x = x_init(seed, n)
    lane_cache: dict[int, np.ndarray] = {}
    warm_e = None
    for t in range(sch.T, sch.T - warmup, -1):
        e = pred(x, t, sch.T)
        _rec(tr, t, x, e, True)
        x = ddpm_step(x, t, e, sch, z_step(seed, t, n))
        warm_e = e
    nbatch = 0
    for cyc in plan_cycles(sch.T, warmup, degree, lengths):
        lanes_in = []
        for j in range(len(cyc)):
            xj = x
            ce = lane_cache.get(j, warm_e)
            for k in range(j):
                xj = ddpm_step(xj, cyc[k], ce, sch, z_step(seed, cyc[k], n))
            lanes_in.append(xj)
        outs = [pred(xj, tj, sch.T) for xj, tj in zip(lanes_in, cyc)]
        nbatch += 1
        for j, tj in enumerate(cyc):
            _rec(tr, tj, x, outs[j], j == 0)
            x = ddpm_step(x, tj, outs[j], sch, z_step(seed, tj, n))
            lane_cache[j] = outs[j]
    tr["x0"] = x
    tr["batch_calls"] = nbatch
    return tr
