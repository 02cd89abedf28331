"""Discrete-event evaluation of a schedule program under the cost model of
PAPER.md §4.2 Table 1 — TEST INFRASTRUCTURE ONLY.

Cost model: per chunk, forward T_F, activation-backward T_B,
weight-backward T_W, TP communication T_AR (same in both directions); PP
communication 0 (Table 1 ignores it; reading Q20).  Block durations (SURVEY
App. A, from §3):
  F      T_F + T_AR              (forward comm cannot be hidden without a braid)
  BFULL  T_B + T_W + max(0, T_AR - T_W)   (backward comm "naturally overlapped"
                                           with W)
  B      T_B + T_AR              (separated backward exposes its comm)
  W      T_W
  FB     T_F + T_B + T_W         (braid, Fig. 3a: every comm hidden)
  FBS    T_F + T_B               (braid, Fig. 3b)
  FW     T_F + T_W
Un-braided expansion (NOBRAID) charges each braided block as its parts run
one after the other; NAIVE charges every backward comm in full.

Execution: each device runs its list in order; an action starts at
max(device free, end of every action it depends on):
  F(mb, vs)  needs F(mb, vs-1);  B(mb, vs) needs B(mb, vs+1) (or F(mb, vs) on
  the last virtual stage);  W(mb, vs) needs B(mb, vs).
Memory (P:L127 M_a per chunk-microbatch): +1 at the start of the action
holding F, -1 at the end of the action that completes its weight gradient
(BFULL/FB end, or W end); frees before allocations at equal times.
"""
from __future__ import annotations

from typing import Dict, List, Tuple

from . import schedule as sc


def block_cost(kind: int, a_kind: int, T_F, T_B, T_W, T_AR):
    """(duration, exposed TP comm) of one action."""
    braid = kind != sc.STP_NOBRAID
    naive = kind == sc.ONEF1B_I_NAIVE
    bfull_exp = T_AR if naive else max(0.0, T_AR - T_W)
    F = (T_F + T_AR, T_AR)
    BF = (T_B + T_W + bfull_exp, bfull_exp)
    B = (T_B + T_AR, T_AR)
    W = (T_W, 0.0)
    if a_kind == sc.A_F:
        return F
    if a_kind == sc.A_BFULL:
        return BF
    if a_kind == sc.A_B:
        return B
    if a_kind == sc.A_W:
        return W
    if a_kind == sc.A_FB:
        return (T_F + T_B + T_W, 0.0) if braid else (F[0] + BF[0], F[1] + BF[1])
    if a_kind == sc.A_FBS:
        return (T_F + T_B, 0.0) if braid else (F[0] + B[0], F[1] + B[1])
    if a_kind == sc.A_FW:
        return (T_F + T_W, 0.0) if braid else (F[0] + W[0], F[1])
    raise ValueError(a_kind)


def _parts(a):
    """(forward mb | None, backward mb | None, backward-is-full, w (mb, chunk) | None)."""
    k, c, f, b, w, wc = a
    fw = f if k in (sc.A_F, sc.A_FB, sc.A_FBS, sc.A_FW) else None
    bw = b if k in (sc.A_BFULL, sc.A_B, sc.A_FB, sc.A_FBS) else None
    full = k in (sc.A_BFULL, sc.A_FB)
    ww = (w, wc) if k in (sc.A_W, sc.A_FW) else None
    return fw, bw, full, ww


def simulate(kind: int, p: int, progs: List[List[tuple]], T_F, T_B, T_W, T_AR):
    V = sc.n_vstages(kind, p)
    fend: Dict[Tuple[int, int], float] = {}     # (mb, vs) -> end time of F
    bend: Dict[Tuple[int, int], float] = {}
    ptr = [0] * p
    free = [0.0] * p
    timeline: List[List[Tuple[float, float]]] = [[] for _ in range(p)]
    exposed = [0.0] * p
    busy = [0.0] * p
    mem_events: List[List[Tuple[float, int]]] = [[] for _ in range(p)]
    total = sum(len(x) for x in progs)
    done = 0
    while done < total:
        progress = False
        for d in range(p):
            while ptr[d] < len(progs[d]):
                a = progs[d][ptr[d]]
                c = a[1]
                fw, bw, full, ww = _parts(a)
                vs = sc.vstage(kind, p, d, c)
                deps = []
                ready = True
                if fw is not None and vs > 0:
                    key = (fw, vs - 1)
                    ready &= key in fend
                    deps.append(fend.get(key, 0.0))
                if bw is not None:
                    key = (bw, vs + 1) if vs < V - 1 else None
                    if key is not None:
                        ready &= key in bend
                        deps.append(bend.get(key, 0.0))
                    ready &= (bw, vs) in fend
                    deps.append(fend.get((bw, vs), 0.0))
                if ww is not None:
                    wvs = sc.vstage(kind, p, d, ww[1])
                    ready &= (ww[0], wvs) in bend
                    deps.append(bend.get((ww[0], wvs), 0.0))
                if not ready:
                    break
                dur, exp = block_cost(kind, a[0], T_F, T_B, T_W, T_AR)
                start = max([free[d]] + deps)
                end = start + dur
                free[d] = end
                timeline[d].append((start, end))
                exposed[d] += exp
                busy[d] += dur
                if fw is not None:
                    fend[(fw, vs)] = end
                    mem_events[d].append((start, +1))
                if bw is not None:
                    bend[(bw, vs)] = end
                    if full:
                        mem_events[d].append((end, -1))
                if ww is not None:
                    mem_events[d].append((end, -1))
                ptr[d] += 1
                done += 1
                progress = True
        if not progress:
            stuck = [(d, progs[d][ptr[d]]) for d in range(p) if ptr[d] < len(progs[d])]
            raise RuntimeError(f"DeadlockDetected: {stuck}")
    makespan = max(free)
    peak = []
    for d in range(p):
        cur = best = 0
        for _, delta in sorted(mem_events[d], key=lambda e: (e[0], e[1])):
            cur += delta
            best = max(best, cur)
        peak.append(best)
    bubble = [makespan - busy[d] for d in range(p)]
    return dict(makespan=makespan, bubble=bubble, exposed=exposed, busy=busy,
                peak=peak, timeline=timeline)


def program_order_peak(kind: int, p: int, d: int, actions) -> int:
    """Max number of chunk-microbatches whose F has been issued but whose
    weight gradient has not, walking the device's list in order (the stash
    slots the executor must hold)."""
    cur = best = 0
    for a in actions:
        fw, bw, full, ww = _parts(a)
        if fw is not None:
            cur += 1
            best = max(best, cur)
        if bw is not None and full:
            cur -= 1
        if ww is not None:
            cur -= 1
    return best


def simulate_durations(kind: int, p: int, progs, durations, pp_latency: float = 0.0):
    """Same dependency semantics as `simulate`, but every action takes the
    given duration (durations[d][i], e.g. measured compute time of action i on
    device d) instead of the Table 1 block cost, and a dependency on an action
    of ANOTHER device arrives pp_latency later (one PP message; Table 1 and
    `simulate` take it as 0, reading Q20).  Returns the makespan — the
    executor-consistency check of SURVEY §8d.4 compares it with the measured
    step time."""
    V = sc.n_vstages(kind, p)
    fend, bend = {}, {}
    ptr = [0] * p
    free = [0.0] * p
    total = sum(len(x) for x in progs)
    done = 0
    while done < total:
        progress = False
        for d in range(p):
            while ptr[d] < len(progs[d]):
                a = progs[d][ptr[d]]
                fw, bw, full, ww = _parts(a)
                vs = sc.vstage(kind, p, d, a[1])
                deps, ready = [], True
                lat = lambda v: pp_latency if sc.vstage_device(kind, p, v)[0] != d else 0.0  # noqa: E731
                if fw is not None and vs > 0:
                    ready &= (fw, vs - 1) in fend
                    deps.append(fend.get((fw, vs - 1), 0.0) + lat(vs - 1))
                if bw is not None:
                    if vs < V - 1:
                        ready &= (bw, vs + 1) in bend
                        deps.append(bend.get((bw, vs + 1), 0.0) + lat(vs + 1))
                    ready &= (bw, vs) in fend
                    deps.append(fend.get((bw, vs), 0.0))
                if ww is not None:
                    wvs = sc.vstage(kind, p, d, ww[1])
                    ready &= (ww[0], wvs) in bend
                    deps.append(bend.get((ww[0], wvs), 0.0))
                if not ready:
                    break
                end = max([free[d]] + deps) + durations[d][ptr[d]]
                free[d] = end
                if fw is not None:
                    fend[(fw, vs)] = end
                if bw is not None:
                    bend[(bw, vs)] = end
                ptr[d] += 1
                done += 1
                progress = True
        if not progress:
            raise RuntimeError("DeadlockDetected")
    return max(free)
