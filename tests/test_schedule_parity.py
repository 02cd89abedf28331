"""The C++ schedule builder + unit expansion (libstp.so, stp_build_schedule /
stp_schedule_serialize) against the independent oracle (oracle/schedule.py):
canonical text must be byte-identical (north_star: "bit-exact for the
schedule and unit order").  CPU only: the library loads without a GPU."""
import ctypes as C

import pytest

from oracle import schedule as sc

GRID = [(k, p, m) for k in (sc.STP, sc.STP_NOSEP, sc.STP_NOBRAID, sc.ZB, sc.ONEF1B_I, sc.ONEF1B_I_NAIVE, sc.ONEF1B,
                            sc.STP_MEM)
        for p in (1, 2, 3, 4, 8) for m in (1, 2, 3, 4, 5, 8, 12, 16, 4 * p + 3)
        if not (k in (sc.ONEF1B_I, sc.ONEF1B_I_NAIVE) and m % p)]


def _L():
    from paper_2510_27257_b200 import _lib
    return _lib


def _cpp_text(kind, p, m, t, lay):
    L = _L()
    v = 1 if kind == sc.ONEF1B else 2
    h = C.c_void_p()
    L.call("stp_build_schedule", p, v, t, m, kind, C.byref(h))
    try:
        arr = (C.c_int32 * len(lay))(*lay) if lay is not None else None
        n = C.c_int64()
        rc = L.lib.stp_schedule_serialize(h, arr, None, 0, C.byref(n))
        assert rc == -8  # STP_ECAPACITY with the needed size
        buf = C.create_string_buffer(n.value + 1)
        L.call("stp_schedule_serialize", h, arr, buf, n.value + 1, C.byref(n))
        return buf.value.decode()
    finally:
        L.lib.stp_free_schedule(h)


def _layers(kind, p, seed):
    V = p if kind == sc.ONEF1B else 2 * p
    return [1 + (seed + i) % 3 for i in range(V)]


@pytest.mark.parametrize("kind,p,m", GRID)
def test_schedule_text_bit_exact(kind, p, m):
    v = 1 if kind == sc.ONEF1B else 2
    assert _cpp_text(kind, p, m, 2, None) == sc.serialize(kind, p, v, 2, m)
    lay = _layers(kind, p, m)
    assert _cpp_text(kind, p, m, 4, lay) == sc.serialize(kind, p, v, 4, m, lay)


def test_errors_and_capacity():
    L = _L()
    h = C.c_void_p()
    assert L.lib.stp_build_schedule(2, 2, 1, 3, sc.ONEF1B_I, C.byref(h)) == -2   # m % p
    assert "n_micro" in L.last_error()
    assert L.lib.stp_build_schedule(2, 3, 1, 4, sc.STP, C.byref(h)) == -2       # vpp != 2
    assert L.lib.stp_build_schedule(0, 2, 1, 4, sc.STP, C.byref(h)) == -1
    L.call("stp_build_schedule", 2, 2, 1, 4, sc.STP, C.byref(h))
    n = C.c_int32()
    assert L.lib.stp_schedule_actions(h, 0, None, 0, C.byref(n)) == -8 and n.value == 15
    buf = (L.Action * n.value)()
    L.call("stp_schedule_actions", h, 0, buf, n.value, C.byref(n))
    got = [sc.action_str((a.kind, a.chunk, a.f_mb, a.b_mb, a.w_mb, a.w_chunk)) for a in buf]
    assert got == [sc.action_str(a) for a in sc.build_program(sc.STP, 2, 4)[0]]
    assert L.lib.stp_schedule_actions(h, 2, buf, n.value, C.byref(n)) == -1
    slots = C.c_int32()
    L.call("stp_schedule_stash_slots", h, 0, C.byref(slots))
    from oracle import simulate as sm
    assert slots.value == sm.program_order_peak(sc.STP, 2, 0, sc.build_program(sc.STP, 2, 4)[0])
    L.lib.stp_free_schedule(h)


def test_layer_split_matches_paper_rule():
    L = _L()
    out = (C.c_int32 * 8)()
    L.call("stp_layer_split", 30, 8, out)
    assert list(out) == [4, 4, 4, 4, 4, 4, 4, 2]
    out4 = (C.c_int32 * 4)()
    L.call("stp_layer_split", 28, 4, out4)
    assert list(out4) == [8, 8, 7, 5]
    assert L.lib.stp_layer_split(8, 8, out) == -1 and "IndivisibleLayers" in L.last_error()


def _cpp_text_mllm(kind, p, m, t, lay):
    L = _L()
    h = C.c_void_p()
    L.call("stp_build_schedule", p, 2, t, m, kind, C.byref(h))
    try:
        arr = (C.c_int32 * len(lay))(*lay)
        n = C.c_int64()
        assert L.lib.stp_schedule_serialize_mllm(h, arr, None, 0, C.byref(n)) == -8
        buf = C.create_string_buffer(n.value + 1)
        L.call("stp_schedule_serialize_mllm", h, arr, buf, n.value + 1, C.byref(n))
        return buf.value.decode()
    finally:
        L.lib.stp_free_schedule(h)


MLLM_GRID = [(k, p, m) for k in (sc.STP, sc.STP_NOSEP, sc.STP_NOBRAID, sc.ZB, sc.ONEF1B_I, sc.STP_MEM)
             for p in (1, 2, 4) for m in (1, 4, 8, 16) if not (k == sc.ONEF1B_I and m % p)]


@pytest.mark.parametrize("kind,p,m", MLLM_GRID)
def test_mllm_schedule_text_bit_exact(kind, p, m):
    """MLLM expansion (ViT layers + merger on vs 0): C++ == oracle, and
    vs 0's lanes carry F_MERGE / B_MERGE / W_MERGE exactly once per microbatch."""
    lay = [3] + [1 + (m + i) % 3 for i in range(2 * p - 1)]
    txt = _cpp_text_mllm(kind, p, m, 2, lay)
    assert txt == sc.serialize(kind, p, 2, 2, m, lay, vit_first=True)
    assert txt.splitlines()[0].endswith(" mllm")
    progs = sc.build_program(kind, p, m)
    d0 = sc.vstage_device(kind, p, 0)[0]
    us = sc.expand_units(kind, p, d0, progs[d0], lay, vit_first=True)
    c0 = sc.vstage_device(kind, p, 0)[1]
    for op in (sc.F_MERGE, sc.B_MERGE, sc.W_MERGE):
        mbs = sorted(u[5] for u in us if u[2] == op)
        assert mbs == list(range(1, m + 1)) and all(u[4] == c0 for u in us if u[2] == op)
    # every ViT layer runs F / B / W once per microbatch on vs 0
    for l in range(lay[0]):
        for op in (sc.F_ATTN, sc.F_MLP, sc.B_ATTN, sc.B_MLP, sc.W_ATTN, sc.W_MLP):
            assert sum(1 for u in us if u[2] == op and u[3] == l) == m
