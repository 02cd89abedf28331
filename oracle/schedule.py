"""Reference schedule builders and the unit expansion of braided execution
blocks — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings:
  R-STP   PAPER.md §4.2 + App. A, Fig. 5 missing:
          1. slot grid, k = 1..m+2p+1, chunk-1 slot then chunk-0 slot
             ("one F&B for model chunk 1, followed by one F&B for chunk 0",
             P:L122): chunk 1 (f = k-p+d, b = k-p-1), chunk 0 (f = k,
             b = k-2p+d); both present -> FB, forward only -> F, backward
             only -> BFULL.
          2. warm-up separation: on every device except d = p-1 ("except for
             the last stage"; Q2) the first p-1 FB become FBS.
          3. degraded separation: every FB after the device's last chunk-0
             forward becomes FBS ("weight separation is reactivated", P:L122;
             Q4).
          4. deferred W (FIFO): F with a non-empty queue -> FW; FBS pushes its
             W; after each BFULL pop one W; the rest at the end ("bubbles are
             filled with stored weight gradient computations"; Q5).
  1F1B-I  Megatron interleaved, v = 2, parallel dataflow vs = c*p + d
          (P:L173): warm-up min(2(p-d-1)+p, 2m) forwards, then F/BFULL
          pairs, then the remaining BFULL.
  1F1B    v = 1 (PipeDream): warm-up min(p-d-1, m) forwards.
  ZB      ZB-V-style greedy (V-shape, every backward split into B and W,
          memory cap 2p chunk-microbatches; priority B > F > W), list-
          scheduled under representative costs (F, B, W) = (12, 15, 9): the
          B200 per-layer unit times at TP4 (F : B : W = 1 : 1.28 : 0.86, plus
          the exposed TP phase of a lone F / B), so its order suits the
          kernels it runs on (round 1 used unit costs; under real costs that
          order left bubbles growing with m).  The exact ZB-V order of Qi et
          al. is not in the paper: PARITY UNPINNED beyond Table 1's closed
          forms (exposure 4m*T_AR, peak 2p).
  NOBRAID R-STP actions, braided actions expanded un-interleaved.
  NOSEP   R-STP slot grid without steps 2-4 (no W separation).
  1F1B-I-NAIVE  1F1B-I actions; every backward W unit waits for the TP
          communication of its own B unit (all TP comm synchronous).
  STP-MEM Ours^, the schedule with the memory-efficient warm-up (App. A
          Fig. 8b, App. B schedule (d); reading R4): V-shape,
          list-scheduled under unit costs with ZB-V's memory budget of 2p
          chunk-microbatches; each decision prefers, in order, a braided
          F(f)&B(b) of one chunk with f > b (App. A: "the microbatch index in
          the forward pass should be greater than that in the backward pass"),
          its weight gradient deferred (FBS, "necessitates decoupling the
          backward pass"); a lone activation backward B; a forward braided with
          the oldest deferred W (FW) or a lone F (the "additional forward pass
          ... before the overlapped F&B execution begins"); a lone W.  Chunk 1
          before chunk 0 at equal readiness.

Unit expansion (Fig. 3) and canonical text
 are defined in DESIGN.md "Unit expansion"; the C++ builder in
paper_2510_27257_b200/csrc/stp_schedule.cpp implements the same definition
independently and must produce identical bytes.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

# schedule kinds (include/stp.h stp_sched_kind)
STP, ONEF1B_I, ZB, STP_NOBRAID, STP_NOSEP, ONEF1B_I_NAIVE, ONEF1B, STP_MEM = range(8)
KIND_NAMES = {STP: "stp", ONEF1B_I: "1f1b-i", ZB: "zb", STP_NOBRAID: "stp-nobraid",
              STP_NOSEP: "stp-nosep", ONEF1B_I_NAIVE: "1f1b-i-naive", ONEF1B: "1f1b", STP_MEM: "stp-mem"}
# action kinds (stp_act_kind)
A_F, A_BFULL, A_B, A_W, A_FB, A_FBS, A_FW = range(7)
ACT_NAMES = ["F", "BFULL", "B", "W", "FB", "FBS", "FW"]
# unit ops (stp_unit_op)
(F_ATTN, F_MLP, B_MLP, B_ATTN, W_MLP, W_ATTN, CF, CB, F_EMB, W_EMB, F_HEAD,
 B_HEAD, W_HEAD, PP_SEND, PP_RECV, F_MERGE, B_MERGE, W_MERGE) = range(18)
S_COMPUTE, S_COMM, S_PP = 0, 1, 2

Action = Tuple[int, int, int, int, int, int]   # kind, chunk, f_mb, b_mb, w_mb, w_chunk


def act(kind, chunk, f=-1, b=-1, w=-1, wc=-1) -> Action:
    return (kind, chunk, f, b, w, wc)


def n_vstages(kind: int, p: int) -> int:
    return p if kind == ONEF1B else 2 * p


def vstage(kind: int, p: int, d: int, c: int) -> int:
    """Virtual stage held by (device d, chunk c)."""
    if kind == ONEF1B:
        return d
    if kind in (ONEF1B_I, ONEF1B_I_NAIVE):
        return c * p + d                      # parallel dataflow
    return d if c == 0 else 2 * p - 1 - d     # V-shape


def vstage_device(kind: int, p: int, vs: int) -> Tuple[int, int]:
    for d in range(p):
        for c in range(1 if kind == ONEF1B else 2):
            if vstage(kind, p, d, c) == vs:
                return d, c
    raise ValueError(vs)


# ---------------------------------------------------------------------------
# builders
# ---------------------------------------------------------------------------

def _rstp_grid(p: int, m: int, d: int) -> List[Action]:
    out = []
    ok = lambda x: 1 <= x <= m
    for k in range(1, m + 2 * p + 2):
        for c, f, b in ((1, k - p + d, k - p - 1), (0, k, k - 2 * p + d)):
            hf, hb = ok(f), ok(b)
            if hf and hb:
                out.append(act(A_FB, c, f, b))
            elif hf:
                out.append(act(A_F, c, f))
            elif hb:
                out.append(act(A_BFULL, c, b=b))
    return out


def build_rstp(p: int, m: int, d: int, separate: bool = True) -> List[Action]:
    acts = _rstp_grid(p, m, d)
    if not separate:
        return acts
    # step 2: warm-up separation on all devices but d = p-1
    if d != p - 1:
        n = 0
        for i, a in enumerate(acts):
            if a[0] == A_FB and n < p - 1:
                acts[i] = (A_FBS,) + a[1:]
                n += 1
    # step 3: degraded separation after the last chunk-0 forward
    last_f0 = max(i for i, a in enumerate(acts) if a[1] == 0 and a[0] in (A_F, A_FB, A_FBS))
    for i in range(last_f0 + 1, len(acts)):
        if acts[i][0] == A_FB:
            acts[i] = (A_FBS,) + acts[i][1:]
    # step 4: deferred-W placement (FIFO)
    queue: List[Tuple[int, int]] = []
    out: List[Action] = []
    for a in acts:
        kind, c, f, b = a[0], a[1], a[2], a[3]
        if kind == A_F and queue:
            wc, wb = queue.pop(0)
            out.append(act(A_FW, c, f, w=wb, wc=wc))
        elif kind == A_FBS:
            out.append(a)
            queue.append((c, b))
        elif kind == A_BFULL:
            out.append(a)
            if queue:
                wc, wb = queue.pop(0)
                out.append(act(A_W, wc, w=wb, wc=wc))
        else:
            out.append(a)
    for wc, wb in queue:
        out.append(act(A_W, wc, w=wb, wc=wc))
    return out


def build_1f1b_interleaved(p: int, m: int, d: int) -> List[Action]:
    if m % p != 0:
        raise ValueError("1F1B-I needs n_micro % pp == 0 (Megatron rule)")
    v = 2
    total = m * v
    nw = min(2 * (p - d - 1) + (v - 1) * p, total)

    def fwd(k):
        c = (k % (p * v)) // p
        return c, (k // (p * v)) * p + (k % p) + 1

    def bwd(k):
        c = v - 1 - (k % (p * v)) // p
        return c, (k // (p * v)) * p + (k % p) + 1

    out = [act(A_F, *fwd(k)) for k in range(nw)]
    for i in range(total - nw):
        c, f = fwd(nw + i)
        out.append(act(A_F, c, f))
        c, b = bwd(i)
        out.append(act(A_BFULL, c, b=b))
    for i in range(total - nw, total):
        c, b = bwd(i)
        out.append(act(A_BFULL, c, b=b))
    return out


def build_1f1b(p: int, m: int, d: int) -> List[Action]:
    nw = min(p - d - 1, m)
    out = [act(A_F, 0, f) for f in range(1, nw + 1)]
    for i in range(m - nw):
        out.append(act(A_F, 0, nw + i + 1))
        out.append(act(A_BFULL, 0, b=i + 1))
    for i in range(m - nw, m):
        out.append(act(A_BFULL, 0, b=i + 1))
    return out


ZB_COSTS = (12, 15, 9)   # (F, B, W) durations of the ZB list schedule (module doc)


def build_zb_greedy(p: int, m: int) -> List[List[Action]]:
    """ZB-V-style greedy list schedule under ZB_COSTS (see module doc)."""
    cF, cB, cW = ZB_COSTS
    V = 2 * p
    cap = 2 * p
    fdone: Dict[Tuple[int, int], int] = {}     # (mb, vs) -> end time
    bdone: Dict[Tuple[int, int], int] = {}
    nextf = [[1, 1] for _ in range(p)]
    nextb = [[1, 1] for _ in range(p)]
    wq: List[List[Tuple[int, int]]] = [[] for _ in range(p)]
    live = [0] * p
    free = [0] * p
    progs: List[List[Action]] = [[] for _ in range(p)]
    total = 3 * 2 * m * p
    t = 0
    n = 0
    while n < total:
        if t > 100 * max(cF, cB, cW) * (total + 10):
            raise RuntimeError("ZB greedy did not terminate")
        for d in range(p):
            if free[d] > t:
                continue
            # B candidates
            choice = None
            for c in (1, 0):
                b = nextb[d][c]
                if b > m:
                    continue
                vs = vstage(ZB, p, d, c)
                dep = (b, vs + 1) if vs < V - 1 else None
                ok = (b, vs) in fdone and fdone[(b, vs)] <= t
                ok = ok and (dep is None or (dep in bdone and bdone[dep] <= t))
                if ok and (choice is None or b < choice[1]):
                    choice = (c, b)
            if choice is not None:
                c, b = choice
                vs = vstage(ZB, p, d, c)
                bdone[(b, vs)] = free[d] = t + cB
                nextb[d][c] += 1
                wq[d].append((c, b))
                progs[d].append(act(A_B, c, b=b))
                n += 1
                continue
            choice = None
            if live[d] < cap:
                for c in (1, 0):
                    f = nextf[d][c]
                    if f > m:
                        continue
                    vs = vstage(ZB, p, d, c)
                    dep = (f, vs - 1) if vs > 0 else None
                    if dep is None or (dep in fdone and fdone[dep] <= t):
                        choice = (c, f)
                        break
            if choice is not None:
                c, f = choice
                vs = vstage(ZB, p, d, c)
                fdone[(f, vs)] = free[d] = t + cF
                nextf[d][c] += 1
                live[d] += 1
                progs[d].append(act(A_F, c, f))
                n += 1
                continue
            if wq[d]:
                c, b = wq[d].pop(0)
                live[d] -= 1
                free[d] = t + cW
                progs[d].append(act(A_W, c, w=b, wc=c))
                n += 1
        t += 1
    return progs


def build_stp_mem(p: int, m: int) -> List[List[Action]]:
    """Ours^ (reading R4, see module doc): unit costs F = B = W = 1 (FBS and
    FW take 2); at every time step each idle device takes the first feasible
    choice in the order FBS > B > FW / F > W."""
    V = 2 * p
    cap = 2 * p
    fend: Dict[Tuple[int, int], int] = {}     # (mb, vs) -> end time
    bend: Dict[Tuple[int, int], int] = {}
    nextf = [[1, 1] for _ in range(p)]
    nextb = [[1, 1] for _ in range(p)]
    wq: List[List[Tuple[int, int]]] = [[] for _ in range(p)]
    live = [0] * p
    free = [0] * p
    progs: List[List[Action]] = [[] for _ in range(p)]
    total = 3 * 2 * m * p
    n = 0
    t = 0

    def f_ready(d, c):
        f = nextf[d][c]
        vs = vstage(STP_MEM, p, d, c)
        return f <= m and (vs == 0 or fend.get((f, vs - 1), total + 1) <= t)

    def b_ready(d, c):
        b = nextb[d][c]
        vs = vstage(STP_MEM, p, d, c)
        if b > m or fend.get((b, vs), total + 1) > t:
            return False
        return vs == V - 1 or bend.get((b, vs + 1), total + 1) <= t

    while n < total:
        if t > 100 * (total + 10):
            raise RuntimeError("STP-MEM list schedule did not terminate")
        for d in range(p):
            if free[d] > t:
                continue
            done = False
            for c in (1, 0):         # braided F&B(separated) of one chunk, f > b
                if (live[d] < cap and b_ready(d, c) and f_ready(d, c)
                        and nextf[d][c] > nextb[d][c]):
                    f, b, vs = nextf[d][c], nextb[d][c], vstage(STP_MEM, p, d, c)
                    fend[(f, vs)] = bend[(b, vs)] = free[d] = t + 2
                    nextf[d][c] += 1
                    nextb[d][c] += 1
                    live[d] += 1
                    wq[d].append((c, b))
                    progs[d].append(act(A_FBS, c, f, b))
                    n += 2
                    done = True
                    break
            if done:
                continue
            for c in (1, 0):         # lone activation backward
                if b_ready(d, c):
                    b, vs = nextb[d][c], vstage(STP_MEM, p, d, c)
                    bend[(b, vs)] = free[d] = t + 1
                    nextb[d][c] += 1
                    wq[d].append((c, b))
                    progs[d].append(act(A_B, c, b=b))
                    n += 1
                    done = True
                    break
            if done:
                continue
            if live[d] < cap:
                for c in (1, 0):     # forward, braided with the oldest deferred W if any
                    if f_ready(d, c):
                        f, vs = nextf[d][c], vstage(STP_MEM, p, d, c)
                        nextf[d][c] += 1
                        live[d] += 1
                        if wq[d]:
                            wc, wb = wq[d].pop(0)
                            live[d] -= 1
                            fend[(f, vs)] = free[d] = t + 2
                            progs[d].append(act(A_FW, c, f, w=wb, wc=wc))
                            n += 2
                        else:
                            fend[(f, vs)] = free[d] = t + 1
                            progs[d].append(act(A_F, c, f))
                            n += 1
                        done = True
                        break
            if done:
                continue
            if wq[d]:
                wc, wb = wq[d].pop(0)
                live[d] -= 1
                free[d] = t + 1
                progs[d].append(act(A_W, wc, w=wb, wc=wc))
                n += 1
        t += 1
    return progs


def build_program(kind: int, p: int, m: int) -> List[List[Action]]:
    """Per-device action lists (Fig. 5 caption: F, B, W per device)."""
    if p < 1 or m < 1:
        raise ValueError("pp >= 1 and n_micro >= 1 required")
    if kind == STP:
        return [build_rstp(p, m, d) for d in range(p)]
    if kind == STP_NOBRAID:
        return [build_rstp(p, m, d) for d in range(p)]
    if kind == STP_NOSEP:
        return [build_rstp(p, m, d, separate=False) for d in range(p)]
    if kind in (ONEF1B_I, ONEF1B_I_NAIVE):
        return [build_1f1b_interleaved(p, m, d) for d in range(p)]
    if kind == ONEF1B:
        return [build_1f1b(p, m, d) for d in range(p)]
    if kind == ZB:
        return build_zb_greedy(p, m)
    if kind == STP_MEM:
        return build_stp_mem(p, m)
    raise ValueError(kind)


# ---------------------------------------------------------------------------
# action text (SURVEY §8c.2 golden notation)
# ---------------------------------------------------------------------------

def action_str(a: Action) -> str:
    kind, c, f, b, w, wc = a
    s = f"{ACT_NAMES[kind]}{c if kind != A_W else wc}"
    if f >= 0:
        s += f" f{f}"
    if b >= 0:
        s += f" b{b}"
    if w >= 0 and kind != A_W:
        s += f" w{w}.{wc}"
    if kind == A_W:
        s += f" w{w}.{wc}"
    return s


# ---------------------------------------------------------------------------
# unit expansion
# ---------------------------------------------------------------------------

class _Emitter:
    def __init__(self):
        self.units: List[Tuple[int, ...]] = []

    def emit(self, action, stream, op, layer, chunk, mb, dep0=-1, dep1=-1) -> int:
        self.units.append((action, stream, op, layer, chunk, mb, dep0, dep1))
        return len(self.units) - 1


def _layers_of(layers_per_vstage: Sequence[int], vs: int) -> List[int]:
    first = sum(layers_per_vstage[:vs])
    return list(range(first, first + layers_per_vstage[vs]))


def expand_units(kind: int, p: int, d: int, actions: List[Action],
                 layers_per_vstage: Sequence[int], vit_first: bool = False) -> List[Tuple[int, ...]]:
    """Expand one device's action list into its unit sequence (emit order =
    host enqueue order).  Tuple fields: action, stream, op, layer, chunk, mb,
    dep0, dep1 (dep = global unit index on this device, -1 = none).

    vit_first (MLLM, "the ViT encoder is assigned to the first virtual
    stage on device 0"; reading V5): virtual stage 0 holds the ViT
    layers 0..layers_per_vstage[0]-1 (the LM layers follow in global
    numbering); its forward lane is F_EMB (patch embedding), the ViT layers'
    F_ATTN / F_MLP, then F_MERGE (2x2 merger + text embedding -> LM input);
    its backward lane starts with B_MERGE and its W list with W_MERGE."""
    V = n_vstages(kind, p)
    assert len(layers_per_vstage) == V
    E = _Emitter()
    fwd_tail: Dict[Tuple[int, int], int] = {}
    bwd_tail: Dict[Tuple[int, int], int] = {}
    braid = kind != STP_NOBRAID
    naive = kind == ONEF1B_I_NAIVE

    def dev_of(vs):
        return vstage_device(kind, p, vs)[0]

    # A lane = dict(pre=[callables], steps=[callables], post=[callables]);
    # each callable emits its units when called (so indices are assigned in
    # emit order).
    def fwd_lane(ai, c, mb):
        vs = vstage(kind, p, d, c)
        L = _layers_of(layers_per_vstage, vs)
        heavy = ([(F_EMB, -1)] if vs == 0 else []) + \
            [u for l in L for u in ((F_ATTN, l), (F_MLP, l))] + \
            ([(F_MERGE, -1)] if vs == 0 and vit_first else []) + \
            ([(F_HEAD, -1)] if vs == V - 1 else [])
        st = {"last": -1}

        def pre():
            rv = -1
            if vs > 0 and dev_of(vs - 1) != d:
                rv = E.emit(ai, S_PP, PP_RECV, dev_of(vs - 1), c, mb)
            if vs > 0:
                st["last"] = E.emit(ai, S_COMM, CF, 0, c, mb, rv)

        def mkstep(k, op, l):
            def step():
                u = E.emit(ai, S_COMPUTE, op, l, c, mb, st["last"])
                st["last"] = E.emit(ai, S_COMM, CF, k, c, mb, u)
            return step

        def post():
            fwd_tail[(c, mb)] = st["last"]
            if vs < V - 1 and dev_of(vs + 1) != d:
                E.emit(ai, S_PP, PP_SEND, dev_of(vs + 1), c, mb, st["last"])

        return [pre], [mkstep(k + 1, op, l) for k, (op, l) in enumerate(heavy)], [post]

    def w_list(vs):
        L = _layers_of(layers_per_vstage, vs)
        return ([(W_HEAD, -1)] if vs == V - 1 else []) + \
            ([(W_MERGE, -1)] if vs == 0 and vit_first else []) + \
            [u for l in reversed(L) for u in ((W_MLP, l), (W_ATTN, l))]

    def bwd_lane(ai, c, mb, with_w):
        vs = vstage(kind, p, d, c)
        L = _layers_of(layers_per_vstage, vs)
        heavy = ([(B_HEAD, -1)] if vs == V - 1 else []) + \
            ([(B_MERGE, -1)] if vs == 0 and vit_first else []) + \
            [u for l in reversed(L) for u in ((B_MLP, l), (B_ATTN, l))]
        wl = w_list(vs)
        st = {"last": -1}

        def pre():
            rv = -1
            if vs < V - 1 and dev_of(vs + 1) != d:
                rv = E.emit(ai, S_PP, PP_RECV, dev_of(vs + 1), c, mb)
            if vs < V - 1:
                st["last"] = E.emit(ai, S_COMM, CB, 0, c, mb, rv)

        def mkstep(k, op, l, wop):
            def step():
                dep = fwd_tail[(c, mb)] if op == B_HEAD else st["last"]
                u = E.emit(ai, S_COMPUTE, op, l, c, mb, dep)
                st["last"] = E.emit(ai, S_COMM, CB, k, c, mb, u)
                if with_w:
                    E.emit(ai, S_COMPUTE, wop[0], wop[1], c, mb, st["last"] if naive else -1)
            return step

        def post():
            bwd_tail[(c, mb)] = st["last"]
            if with_w and vs == 0:
                E.emit(ai, S_COMPUTE, W_EMB, -1, c, mb, st["last"])
            if vs > 0 and dev_of(vs - 1) != d:
                E.emit(ai, S_PP, PP_SEND, dev_of(vs - 1), c, mb, st["last"])

        steps = [mkstep(k + 1, op, l, wl[k]) for k, (op, l) in enumerate(heavy)]
        return [pre], steps, [post]

    def w_lane(ai, c, mb):
        vs = vstage(kind, p, d, c)
        wl = w_list(vs)

        def mkstep(op, l):
            return lambda: E.emit(ai, S_COMPUTE, op, l, c, mb)

        def post():
            if vs == 0:
                E.emit(ai, S_COMPUTE, W_EMB, -1, c, mb, bwd_tail[(c, mb)])

        return [], [mkstep(op, l) for op, l in wl], [post]

    def run(lanes, interleave):
        if interleave:
            for ln in lanes:
                for f in ln[0]:
                    f()
            n = max(len(ln[1]) for ln in lanes)
            for k in range(n):
                for ln in lanes:
                    if k < len(ln[1]):
                        ln[1][k]()
            for ln in lanes:
                for f in ln[2]:
                    f()
        else:
            for ln in lanes:
                for f in ln[0] + ln[1] + ln[2]:
                    f()

    for ai, a in enumerate(actions):
        kind_a, c, f, b, w, wc = a
        if kind_a == A_F:
            run([fwd_lane(ai, c, f)], True)
        elif kind_a == A_BFULL:
            run([bwd_lane(ai, c, b, True)], True)
        elif kind_a == A_B:
            run([bwd_lane(ai, c, b, False)], True)
        elif kind_a == A_W:
            run([w_lane(ai, wc, w)], True)
        elif kind_a == A_FB:
            run([fwd_lane(ai, c, f), bwd_lane(ai, c, b, True)], braid)
        elif kind_a == A_FBS:
            run([fwd_lane(ai, c, f), bwd_lane(ai, c, b, False)], braid)
        elif kind_a == A_FW:
            run([fwd_lane(ai, c, f), w_lane(ai, wc, w)], braid)
        else:
            raise ValueError(a)
    return E.units


# ---------------------------------------------------------------------------
# canonical serialisation
# ---------------------------------------------------------------------------

def serialize(kind: int, p: int, v: int, t: int, m: int,
              layers_per_vstage: Optional[Sequence[int]] = None, vit_first: bool = False) -> str:
    progs = build_program(kind, p, m)
    lines = [f"sched {KIND_NAMES[kind]} p {p} v {v} t {t} m {m}" + (" mllm" if vit_first else "")]
    for d, acts in enumerate(progs):
        lines.append(f"rank {d}")
        for i, a in enumerate(acts):
            lines.append("A " + " ".join(str(x) for x in (i,) + a))
        if layers_per_vstage is not None:
            for j, u in enumerate(expand_units(kind, p, d, acts, layers_per_vstage, vit_first)):
                lines.append("U " + " ".join(str(x) for x in (j,) + u))
    return "\n".join(lines) + "\n"


def paper_layer_split(n_layers: int, n_slots: int) -> List[int]:
    """Layers per virtual-stage slot in V order (reading Q17).

    Spread L+2 as evenly as possible (remainder to the earliest slots), then
    take 2 from the last slot.  (The product's copy is stp_layer_split in csrc/schedule.cpp; they share
    no code.)
    """
    total = n_layers + 2
    base, rem = divmod(total, n_slots)
    split = [base + (1 if i < rem else 0) for i in range(n_slots)]
    split[-1] -= 2
    if min(split) < 1 or sum(split) != n_layers:
        raise ValueError(f"IndivisibleLayers: {n_layers} layers over {n_slots} slots")
    return split
