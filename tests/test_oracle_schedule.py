"""Pins for oracle/schedule.py and oracle/simulate.py.

External pins (each is fixed by PAPER.md or textbook pipeline math, not by
the oracle itself):
  * Table 1 closed forms: 1F1B-I PP bubble and TP bubble exact;
    R-STP TP bubble (2p+1)*T_AR and peak 3p*M_a exact; ZB-V TP bubble
    4m*T_AR and peak 2p; R-STP bubble "approximate" -> makespan within 12%
    of the closed-form makespan for m >= 4p (reading Q8).
  * plain 1F1B (PipeDream): the textbook bubble (p-1)(T_F+T_B+T_W).
  * §4.2 text: first braid F(2)&B(1); separation off in the
    steady phase; App. A: forward mb > backward mb in every braid.
  * Table 5 memory ratios.
  * SURVEY §8c.2 golden lists (tests/golden/rstp_survey_8c2.txt).
Invariants over a grid: completeness, F < B < W, no deadlock.
"""
import os

import pytest

from oracle import schedule as sc
from oracle import simulate as sm

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "rstp_survey_8c2.txt")
KINDS = {"stp": sc.STP, "1f1b-i": sc.ONEF1B_I}


def _golden():
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        head, body = line.split(":", 1)
        name, pp, mm, dev = head.split()
        yield KINDS[name], int(pp[2:]), int(mm[2:]), int(dev[3:]), body.strip()


@pytest.mark.parametrize("case", list(_golden()), ids=lambda c: f"{c[0]}-{c[1]}-{c[2]}-{c[3]}")
def test_golden_action_lists(case):
    kind, p, m, d, text = case
    got = " | ".join(sc.action_str(a) for a in sc.build_program(kind, p, m)[d])
    assert got == text


COSTS = [(4, 4, 2, 1), (4, 4, 4, 0), (10, 12, 8, 4), (3, 5, 4, 2)]


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("mult", [1, 2, 4])
@pytest.mark.parametrize("costs", COSTS)
def test_1f1b_interleaved_table1_exact(p, mult, costs):
    T_F, T_B, T_W, T_AR = costs
    m = mult * p
    r = sm.simulate(sc.ONEF1B_I, p, sc.build_program(sc.ONEF1B_I, p, m), T_F, T_B, T_W, T_AR)
    for d in range(p):
        assert r["bubble"][d] == (p - 1) * (T_F + T_AR + T_B + T_W)      # Table 1 row 1
        assert r["exposed"][d] == 2 * m * T_AR if T_W >= T_AR else True  # Table 1 TP col
    # peak (3p-2)*M_a of Table 1 under its counting; ours counts F-start..B-end (Q7)
    if m >= 2 * p:
        assert r["peak"][0] in (3 * p - 2, 3 * p - 1)


@pytest.mark.parametrize("p", [1, 2, 4, 8])
@pytest.mark.parametrize("m", [1, 3, 8, 16])
def test_plain_1f1b_textbook_bubble(p, m):
    T_F, T_B, T_W = 3, 5, 2
    r = sm.simulate(sc.ONEF1B, p, sc.build_program(sc.ONEF1B, p, m), T_F, T_B, T_W, 0)
    for d in range(p):
        assert r["bubble"][d] == (p - 1) * (T_F + T_B + T_W)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("costs", [(10, 12, 8, 4), (4, 4, 2, 1), (6, 9, 6, 6)])
def test_rstp_table1_tp_bubble_and_peak(p, costs):
    T_F, T_B, T_W, T_AR = costs
    for m in (4 * p, 6 * p, 8 * p):
        r = sm.simulate(sc.STP, p, sc.build_program(sc.STP, p, m), T_F, T_B, T_W, T_AR)
        assert max(r["exposed"]) == (2 * p + 1) * T_AR     # Table 1 "Ours" TP column
        # Table 1 "Ours" memory; p = 1 is degenerate (both chunks on one device: 3p+1)
        assert max(r["peak"]) == (3 * p if p > 1 else 4)
        closed = 2 * m * (T_F + T_B + T_W) + (p - 1) * (T_F + T_AR + T_B - T_W) + (2 * p + 1) * T_AR
        assert closed <= r["makespan"] <= 1.12 * closed     # "approximate bubble size" (Q8)


@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_rstp_beats_1f1b_interleaved(p):
    for m in (4 * p, 8 * p):
        for costs in ((10, 12, 8, 4), (4, 4, 2, 1)):
            a = sm.simulate(sc.STP, p, sc.build_program(sc.STP, p, m), *costs)
            b = sm.simulate(sc.ONEF1B_I, p, sc.build_program(sc.ONEF1B_I, p, m), *costs)
            assert a["makespan"] < b["makespan"]


def test_table1_arithmetic_examples():
    # SPEC S:L363-365 evaluates Table 1 at p=4, T_F=4, T_AR=1, T_B=4, T_W=2
    p, T_F, T_AR, T_B, T_W, m = 4, 4, 1, 4, 2, 12
    r = sm.simulate(sc.ONEF1B_I, p, sc.build_program(sc.ONEF1B_I, p, m), T_F, T_B, T_W, T_AR)
    assert r["bubble"][0] == 33 and r["exposed"][0] == 24
    r = sm.simulate(sc.STP, p, sc.build_program(sc.STP, p, m), T_F, T_B, T_W, T_AR)
    assert max(r["exposed"]) == 9 and max(r["peak"]) == 12
    r = sm.simulate(sc.ZB, p, sc.build_program(sc.ZB, p, m), T_F, T_B, T_W, T_AR)
    assert max(r["exposed"]) == 48 and max(r["peak"]) == 8


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_zb_closed_forms(p):
    for m in (2 * p, 4 * p):
        progs = sc.build_program(sc.ZB, p, m)
        assert not any(a[0] == sc.A_BFULL for pr in progs for a in pr)
        r = sm.simulate(sc.ZB, p, progs, 10, 12, 8, 4)
        assert all(e == 4 * m * 4 for e in r["exposed"])    # Table 1 ZB-V TP column
        assert max(r["peak"]) <= 2 * p                      # Table 1 ZB-V memory


def test_table5_memory_ratios():
    # Table 5: 1F1B-I / ZB-V peak = 41/30 at p=4 and 55/38 at p=8;
    # STP / ZB-V = 54/30 at p=4 once App. C's ~+19% per-microbatch overhead (P:L637,
    # 4.3/3.6) is applied to the schedule-level 3p / 2p.
    for p, paper in ((4, 41 / 30), (8, 55 / 38)):
        m = 4 * p
        a = max(sm.simulate(sc.ONEF1B_I, p, sc.build_program(sc.ONEF1B_I, p, m), 4, 4, 2, 1)["peak"])
        b = max(sm.simulate(sc.ZB, p, sc.build_program(sc.ZB, p, m), 4, 4, 2, 1)["peak"])
        assert abs(a / b - paper) / paper < 0.02
    p = 4
    s = max(sm.simulate(sc.STP, p, sc.build_program(sc.STP, p, 16), 4, 4, 2, 1)["peak"])
    b = max(sm.simulate(sc.ZB, p, sc.build_program(sc.ZB, p, 16), 4, 4, 2, 1)["peak"])
    assert abs(s / b * (4.3 / 3.6) - 54 / 30) / (54 / 30) < 0.02


def _check_program(kind, p, m, progs):
    V = sc.n_vstages(kind, p)
    F, B, W = {}, {}, {}
    for d, acts in enumerate(progs):
        for i, a in enumerate(acts):
            k, c, f, b, w, wc = a
            if k in (sc.A_F, sc.A_FB, sc.A_FBS, sc.A_FW):
                key = (f, sc.vstage(kind, p, d, c))
                assert key not in F
                F[key] = (d, i)
            if k in (sc.A_BFULL, sc.A_FB, sc.A_B, sc.A_FBS):
                key = (b, sc.vstage(kind, p, d, c))
                assert key not in B
                B[key] = (d, i)
                if k in (sc.A_BFULL, sc.A_FB):
                    W[key] = (d, i)
            if k in (sc.A_W, sc.A_FW):
                key = (w, sc.vstage(kind, p, d, wc))
                assert key not in W
                W[key] = (d, i)
            if k in (sc.A_FB, sc.A_FBS):
                assert f > b                                # App. A rule
    want = {(mb, vs) for mb in range(1, m + 1) for vs in range(V)}
    assert set(F) == want and set(B) == want and set(W) == want
    for key in want:
        assert F[key][0] == B[key][0] == W[key][0]
        assert F[key][1] <= B[key][1] <= W[key][1]
        if F[key][1] == B[key][1]:
            pytest.fail("F and B of the same (mb, vs) in one action")


@pytest.mark.parametrize("kind", [sc.STP, sc.STP_NOSEP, sc.ONEF1B_I, sc.ZB, sc.ONEF1B, sc.STP_MEM])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 8])
def test_program_invariants_and_no_deadlock(kind, p):
    for m in range(1, 4 * p + 5):
        if kind in (sc.ONEF1B_I,) and m % p:
            with pytest.raises(ValueError):
                sc.build_program(kind, p, m)
            continue
        progs = sc.build_program(kind, p, m)
        _check_program(kind, p, m, progs)
        sm.simulate(kind, p, progs, 10, 12, 8, 4)          # raises on deadlock


@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_rstp_phase_claims(p):
    m = 4 * p
    progs = sc.build_program(sc.STP, p, m)
    for d, acts in enumerate(progs):
        braids = [a for a in acts if a[0] in (sc.A_FB, sc.A_FBS)]
        if d == 0:   # device 0 opens with "the first and second microbatches"
            assert (braids[0][2], braids[0][3]) == (2, 1)
        assert braids[0][3] == 1
        # steady phase: separation deactivated while new microbatches arrive
        last_f0 = max(i for i, a in enumerate(acts) if a[1] == 0 and a[0] in (sc.A_F, sc.A_FB, sc.A_FBS, sc.A_FW))
        warm = p - 1 if d != p - 1 else 0
        sep_before = [a for a in acts[:last_f0 + 1] if a[0] == sc.A_FBS]
        assert len(sep_before) == warm
        if d == p - 1:
            assert not sep_before                           # "except for the last stage"
    first = next(a for a in progs[0] if a[0] in (sc.A_FB, sc.A_FBS))
    assert sc.action_str(first) == "FBS1 f2 b1"


@pytest.mark.parametrize("kind", [sc.STP, sc.STP_NOBRAID, sc.ONEF1B_I, sc.ONEF1B_I_NAIVE, sc.ZB, sc.STP_MEM])
@pytest.mark.parametrize("p,lay", [(1, [2, 1]), (2, [1, 1, 1, 1]), (2, [2, 1, 2, 1]), (3, [1] * 6)])
def test_unit_expansion_invariants(kind, p, lay):
    m = 2 * p
    progs = sc.build_program(kind, p, m)
    for d, acts in enumerate(progs):
        units = sc.expand_units(kind, p, d, acts, lay)
        seen = {}
        for j, u in enumerate(units):
            ai, stream, op, layer, c, mb, d0, d1 = u
            assert 0 <= ai < len(acts)
            assert d0 < j and d1 < j
            if op in (sc.F_ATTN, sc.F_MLP, sc.B_MLP, sc.B_ATTN, sc.W_MLP, sc.W_ATTN,
                      sc.F_EMB, sc.W_EMB, sc.F_HEAD, sc.B_HEAD, sc.W_HEAD):
                assert stream == sc.S_COMPUTE
                key = (op, layer, c, mb)
                assert key not in seen
                seen[key] = j
            elif op in (sc.CF, sc.CB):
                assert stream == sc.S_COMM
            else:
                assert stream == sc.S_PP
        # every layer's six heavy units per (mb, chunk) exactly once
        for c in range(1 if kind == sc.ONEF1B else 2):
            vs = sc.vstage(kind, p, d, c)
            first = sum(lay[:vs])
            for mb in range(1, m + 1):
                for l in range(first, first + lay[vs]):
                    for op in (sc.F_ATTN, sc.F_MLP, sc.B_MLP, sc.B_ATTN, sc.W_MLP, sc.W_ATTN):
                        assert (op, l, c, mb) in seen
                # W after B after F
                l = first
                assert seen[(sc.F_ATTN, l, c, mb)] < seen[(sc.B_ATTN, l, c, mb)] < seen[(sc.W_ATTN, l, c, mb)]


def test_fb_braid_alternates_forward_and_backward():
    # Fig. 3a: compute stream alternates F units of mb f and B units of mb b
    p, lay = 1, [2, 2]
    acts = sc.build_program(sc.STP, p, 3)[0]
    ai = next(i for i, a in enumerate(acts) if a[0] == sc.A_FB)
    units = [u for u in sc.expand_units(sc.STP, p, 0, acts, lay) if u[0] == ai and u[1] == sc.S_COMPUTE]
    ops = [u[2] for u in units]
    fwd = {sc.F_ATTN, sc.F_MLP, sc.F_EMB, sc.F_HEAD}
    pattern = ["f" if o in fwd else ("b" if o in (sc.B_MLP, sc.B_ATTN, sc.B_HEAD) else "w") for o in ops]
    assert "".join(pattern).startswith("fbwfbwfbwfbw")


def test_serialize_header_and_shape():
    txt = sc.serialize(sc.STP, 2, 2, 2, 4, [1, 1, 1, 1])
    lines = txt.split("\n")
    assert lines[0] == "sched stp p 2 v 2 t 2 m 4"
    assert lines[1] == "rank 0"
    assert lines[2] == "A 0 0 0 1 -1 -1 -1"
    assert txt.endswith("\n")


def test_simulated_8gpu_rows_from_measured_units():
    """the simulated TP4 x PP2 rows (tests/simulate_8gpu.py, fed with
    unit times measured on 4x B200) run, and the braid hides TP comm there:
    STP's exposed TP stays below 1F1B-I's and well below the naive schedule's."""
    import json
    import os
    from tests import simulate_8gpu
    prof = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
    stp = json.load(open(os.path.join(prof, "r01_unit_times_tp4_stp.json")))["units"]
    ref = json.load(open(os.path.join(prof, "r01_unit_times_tp4_1f1b-i.json")))["units"]
    res = simulate_8gpu.run(stp, ref, ms=(8, 16))
    for row in res["rows"]:
        assert row["stp"]["exposed_tp_pct"] < row["1f1b-i"]["exposed_tp_pct"] < row["1f1b-i-naive"]["exposed_tp_pct"]
        assert row["stp"]["peak_chunks"] == 6  # 3p
        assert 0.8 < row["stp_vs_1f1b_i"] < 1.3


# ---------------------------------------------------------------------------
# simulate_durations / program_order_peak pins (VERDICT r1 "unpinned oracle parts")

ALL_KINDS = [sc.STP, sc.ONEF1B_I, sc.ZB, sc.STP_NOBRAID, sc.STP_NOSEP, sc.ONEF1B_I_NAIVE, sc.STP_MEM]


@pytest.mark.parametrize("kind", ALL_KINDS)
@pytest.mark.parametrize("p,m", [(1, 3), (2, 4), (2, 8), (4, 8), (4, 16), (8, 16)])
def test_simulate_durations_reproduces_block_costs(kind, p, m):
    """Fed the Table 1 block cost of every action, the duration-driven
    simulator must reproduce simulate()'s makespan exactly (same dependency
    semantics, P:L124-148 cost model)."""
    if kind in (sc.ONEF1B_I, sc.ONEF1B_I_NAIVE) and m % p:
        pytest.skip("1F1B-I needs m % p == 0")
    progs = sc.build_program(kind, p, m)
    costs = (10.0, 12.0, 8.0, 4.0)
    r = sm.simulate(kind, p, progs, *costs)
    durs = [[sm.block_cost(kind, a[0], *costs)[0] for a in progs[d]] for d in range(p)]
    assert sm.simulate_durations(kind, p, progs, durs) == pytest.approx(r["makespan"], rel=0, abs=1e-9)


@pytest.mark.parametrize("kind", [sc.STP, sc.ZB, sc.STP_NOSEP])
@pytest.mark.parametrize("m", [1, 3, 8])
def test_simulate_durations_single_device_is_the_sum(kind, m):
    """p = 1: every dependency is satisfied by program order, so the device
    never idles and the makespan is the plain sum of the action durations."""
    progs = sc.build_program(kind, 1, m)
    durs = [[1.0 + 0.37 * i for i in range(len(progs[0]))]]
    assert sm.simulate_durations(kind, 1, progs, durs) == pytest.approx(sum(durs[0]), abs=1e-9)


@pytest.mark.parametrize("p,mult", [(2, 1), (2, 3), (4, 2), (8, 1)])
def test_simulate_durations_1f1b_interleaved_closed_form(p, mult):
    """Megatron 1F1B-I with per-chunk costs (T_F, T_B+T_W) and no TP comm:
    makespan = 2m (T_F + T_B + T_W) + (p - 1)(T_F + T_B + T_W) (Table 1's
    1F1B-I PP bubble, with T_AR = 0)."""
    m = mult * p
    progs = sc.build_program(sc.ONEF1B_I, p, m)
    TF, TB, TW = 3.0, 4.0, 2.0
    durs = [[TF if a[0] == sc.A_F else TB + TW for a in progs[d]] for d in range(p)]
    assert sm.simulate_durations(sc.ONEF1B_I, p, progs, durs) == pytest.approx(
        2 * m * (TF + TB + TW) + (p - 1) * (TF + TB + TW), abs=1e-9)


@pytest.mark.parametrize("kind", ALL_KINDS)
@pytest.mark.parametrize("p,m", [(2, 4), (2, 16), (4, 8), (4, 32), (8, 32)])
def test_program_order_peak_equals_simulated_peak(kind, p, m):
    """A device runs its list sequentially, so the stash count walked in
    program order must equal the time-based peak of the simulator (alloc at
    an F's action start, free at the end of the action completing its W)."""
    if kind in (sc.ONEF1B_I, sc.ONEF1B_I_NAIVE) and m % p:
        pytest.skip("1F1B-I needs m % p == 0")
    progs = sc.build_program(kind, p, m)
    r = sm.simulate(kind, p, progs, 10.0, 12.0, 8.0, 4.0)
    for d in range(p):
        assert sm.program_order_peak(kind, p, d, progs[d]) == r["peak"][d]


@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_program_order_peak_table1_memory(p):
    """Table 1 memory column: Ours 3p·M_a (exact, max over
    devices), ZB-V at most 2p, 1F1B-I 3p-1 under the F-start..W-end counting
    (reading Q7)."""
    m = 4 * p
    peak = lambda kind: max(sm.program_order_peak(kind, p, d, x)
                            for d, x in enumerate(sc.build_program(kind, p, m)))
    assert peak(sc.STP) == 3 * p
    assert peak(sc.ZB) <= 2 * p
    assert peak(sc.ONEF1B_I) in (3 * p - 2, 3 * p - 1)


def test_paper_layer_split():
    """'the last stage has two fewer layers' for the 152,064 vocab;
    reading Q17 for non-divisible splits."""
    assert sc.paper_layer_split(28, 4) == [8, 8, 7, 5]
    assert sc.paper_layer_split(48, 8) == [7, 7, 6, 6, 6, 6, 6, 4]
    assert sc.paper_layer_split(28, 3) == [10, 10, 8]
    assert sc.paper_layer_split(30, 8) == [4, 4, 4, 4, 4, 4, 4, 2]
    with pytest.raises(ValueError):
        sc.paper_layer_split(8, 8)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_simulate_durations_pp_latency_plain_1f1b(p):
    """Plain 1F1B (one chunk per device), forward / backward costs F, B and a
    message latency c on every stage boundary.  One microbatch is a single
    dependency path: F on devices 0..p-1, then B on p-1..0, with 2(p-1)
    messages, so makespan = p (F + B) + 2 (p - 1) c exactly; with m
    microbatches the latency can only add time, and at c = 0 the textbook
    m (F + B) + (p - 1)(F + B) holds."""
    F, B, c = 3.0, 5.0, 0.7
    progs = sc.build_program(sc.ONEF1B, p, 1)
    durs = [[F if a[0] == sc.A_F else B for a in progs[d]] for d in range(p)]
    assert sm.simulate_durations(sc.ONEF1B, p, progs, durs, pp_latency=c) == pytest.approx(
        p * (F + B) + 2 * (p - 1) * c)
    m = 2 * p
    progs = sc.build_program(sc.ONEF1B, p, m)
    durs = [[F if a[0] == sc.A_F else B for a in progs[d]] for d in range(p)]
    base = sm.simulate_durations(sc.ONEF1B, p, progs, durs)
    assert base == pytest.approx(m * (F + B) + (p - 1) * (F + B))
    assert sm.simulate_durations(sc.ONEF1B, p, progs, durs, pp_latency=c) >= base + 2 * (p - 1) * c - 1e-9


# ---------------------------------------------------------------------------
# Ours^ (STP-MEM, reading R4): the paper's claims about schedule (d)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
def test_stp_mem_app_a_braids_and_separation(p):
    """App. A: every overlapped F&B pairs a forward microbatch index
    greater than the backward one, the backward is decoupled from W (FBS, no FB
    / BFULL), and each chunk's first action on a device is a lone forward (the
    'additional forward pass ... before the overlapped F&B execution')."""
    m = 4 * p
    for d, acts in enumerate(sc.build_program(sc.STP_MEM, p, m)):
        assert not [a for a in acts if a[0] in (sc.A_FB, sc.A_BFULL)]
        assert all(a[2] > a[3] for a in acts if a[0] == sc.A_FBS)
        for c in (0, 1):
            first = next(a for a in acts if a[1] == c and a[0] != sc.A_W)
            assert first[0] in (sc.A_F, sc.A_FW) and first[2] == 1


@pytest.mark.parametrize("p,m", [(2, 8), (2, 16), (4, 12), (4, 16), (4, 32), (8, 32)])
def test_stp_mem_app_b_memory_and_bubbles(p, m):
    """App. B: schedule (d) 'has a lower peak memory footprint
    compared to our standard schedule (c)' -- at most ZB-V's 2p (Table 1) vs
    Ours' 3p -- 'it introduces additional PP bubbles' (longer makespan than
    (c) under the Table 1 cost model) and it still hides part of the TP
    communication ('large TP overheads'): less exposed than ZB-V's 4m T_AR."""
    costs = (10.0, 12.0, 8.0, 4.0)
    mem = sm.simulate(sc.STP_MEM, p, sc.build_program(sc.STP_MEM, p, m), *costs)
    ours = sm.simulate(sc.STP, p, sc.build_program(sc.STP, p, m), *costs)
    assert max(mem["peak"]) <= 2 * p < max(ours["peak"]) == 3 * p
    assert mem["makespan"] > ours["makespan"]
    assert max(mem["exposed"]) < 4 * m * costs[3]
