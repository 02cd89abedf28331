"""8-GPU rows are SIMULATED (gpurun grants <= 4 GPUs): the
oracle's discrete-event simulator of the Table-1 cost model (§4.2,
P:L124-148) fed with per-unit times MEASURED on 4x B200 (TP=4, Qwen2-7B
shape, seq 6144; profiles/r01_unit_times_tp4_{stp,1f1b-i}.json, written by
tools/comm_phase_times.py).  The simulated grid is TP=4 x PP=2 (8 GPUs),
whose per-rank units have exactly the measured TP=4 shapes; only the PP
degree differs.  Per chunk of L_c = 28 / (p * v) = 7 layers:

  T_F  = L_c * (F_ATTN + F_MLP)     T_B = L_c * (B_ATTN + B_MLP)
  T_W  = L_c * (W_ATTN + W_MLP)     T_AR = L_c * 2 * (mean forward comm phase)

with the compute costs of the 1F1B-I run (no overlapped comm: uncontended)
and of the STP run (comm overlapped: includes the measured contention), and
T_AR from 1F1B-I's comm phases (not overlapped: their duration is the
transfer).  PP messages cost 0 (Table 1; our PP sends run on their own
streams).  Embedding / LM head are left out (both schedules pay them once).

Test infrastructure (imports oracle/); run:  python tests/simulate_8gpu.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import schedule as sc  # noqa: E402
from oracle import simulate as sm  # noqa: E402

SEQ = 6144


def per_layer(units):
    u = {k: v["mean_ms"] for k, v in units.items()}
    return (u["F_ATTN"] + u["F_MLP"], u["B_ATTN"] + u["B_MLP"], u["W_ATTN"] + u["W_MLP"], 2 * u["CF"])


def run(stp_units, ref_units, p=2, layers=28, ms=(8, 16, 32)):
    Lc = layers / (2 * p)
    f_s, b_s, w_s, _ = per_layer(stp_units)
    f_r, b_r, w_r, ar = per_layer(ref_units)
    out = {"grid": f"tp4 x pp{p} (8 GPUs, simulated)", "L_c": Lc,
           "per_layer_ms": {"stp": [f_s, b_s, w_s], "1f1b-i": [f_r, b_r, w_r], "T_AR_per_layer": ar}, "rows": []}
    for m in ms:
        row = {"m": m}
        for name, kind, (f, b, w) in (("stp", sc.STP, (f_s, b_s, w_s)),
                                      ("stp_uncontended", sc.STP, (f_r, b_r, w_r)),
                                      ("1f1b-i", sc.ONEF1B_I, (f_r, b_r, w_r)),
                                      ("1f1b-i-naive", sc.ONEF1B_I_NAIVE, (f_r, b_r, w_r))):
            if kind in (sc.ONEF1B_I, sc.ONEF1B_I_NAIVE) and m % p:
                continue
            r = sm.simulate(kind, p, sc.build_program(kind, p, m), Lc * f, Lc * b, Lc * w, Lc * ar)
            row[name] = {"makespan_ms": r["makespan"], "tokens_per_s": m * SEQ / (r["makespan"] / 1e3),
                         "exposed_tp_pct": 100 * max(r["exposed"]) / r["makespan"],
                         "bubble_pct": 100 * max(r["bubble"]) / r["makespan"], "peak_chunks": max(r["peak"])}
        row["stp_vs_1f1b_i"] = row["stp"]["tokens_per_s"] / row["1f1b-i"]["tokens_per_s"]
        out["rows"].append(row)
    return out


def load_units(path):
    """tools/comm_phase_times.py output: one JSON document, possibly after
    NCCL's version banner (round 2) or pretty-printed (round 1)."""
    text = open(path).read()
    return json.loads(text[text.index("{"):])


def main():
    """python tests/simulate_8gpu.py [OUT.json [STP_UNITS.json REF_UNITS.json]]
    (default: the round-1 unit times)."""
    prof = os.path.join(ROOT, "profiles")
    if len(sys.argv) > 3:
        stp_path, ref_path = sys.argv[2], sys.argv[3]
    else:
        stp_path = os.path.join(prof, "r01_unit_times_tp4_stp.json")
        ref_path = os.path.join(prof, "r01_unit_times_tp4_1f1b-i.json")
    stp, ref = load_units(stp_path), load_units(ref_path)
    res = run(stp["units"], ref["units"])
    res["label"] = "SIMULATED (oracle simulator, measured TP=4 unit times) - not a measurement"
    res["unit_times"] = {"stp": os.path.relpath(stp_path, ROOT) + f" ({stp.get('sched')}, {stp.get('transport')})",
                         "reference": os.path.relpath(ref_path, ROOT) + f" ({ref.get('sched')}, {ref.get('transport')})"}
    print(json.dumps(res, indent=1))
    if len(sys.argv) > 1:
        json.dump(res, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
