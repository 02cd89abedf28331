"""libstp.so loads on a CPU-only box and exports every function declared in
include/stp.h and include/stp_ops.h (no compute calls: no GPU here)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("stp.h", "stp_ops.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"\b(stp_[a-z0-9_]+)\s*\(", txt):
            names.add(m.group(1))
    return names


def test_every_declared_symbol_is_exported():
    from paper_2510_27257_b200 import _lib
    names = _declared()
    assert len(names) > 40
    missing = [n for n in sorted(names) if not hasattr(_lib.lib, n)]
    assert not missing, missing
    assert not _lib.MISSING


def test_host_only_calls_work_without_gpu():
    from paper_2510_27257_b200 import _lib
    assert _lib.lib.stp_version().decode().startswith("stp-b200")
    assert _lib.lib.stp_nccl_id_bytes() == 128
    assert _lib.lib.stp_op_attn_bwd_ws_bytes(10, 2, 1, 64) == 80
    # error path: invalid args report through stp_last_error
    assert _lib.lib.stp_build_schedule(0, 2, 1, 1, 0, None) == -1
    assert "out is NULL" in _lib.last_error() or "pp" in _lib.last_error()
