"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
bench.py over one training step: the window runs from the first embedding
launch of step k to that of step k+1 (m embedding launches per step).

    python tools/launch_summary.py LAUNCHES.csv[.gz] --m 8 [--step 1]
"""
import argparse
import collections
import csv
import gzip
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--m", type=int, default=8)
    ap.add_argument("--step", type=int, default=1, help="0-based step index (0 = first warm-up step)")
    a = ap.parse_args()
    op = gzip.open if a.csv.endswith(".gz") else open
    rows = list(csv.reader(op(a.csv, "rt")))
    i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[i], rows[i + 1:]
    ik, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
    seq = []
    for r in data:
        if len(r) <= iv:
            continue
        name = re.sub(r"\(.*", "", r[ik])
        name = re.sub(r"stp::|<unnamed>::|\(anonymous namespace\)::|void ", "", name).strip()
        seq.append((int(r[iid]), name, float(r[iv].replace(",", "")) / 1e6))  # ns -> ms
    emb = [k for k, (_, n, _) in enumerate(seq) if n.startswith("embed_fwd_kernel")]
    starts = emb[::a.m]
    lo, hi = starts[a.step], starts[a.step + 1] if a.step + 1 < len(starts) else len(seq)
    win = seq[lo:hi]
    tot = sum(t for _, _, t in win)
    agg, cnt = collections.defaultdict(float), collections.Counter()
    for _, n, t in win:
        agg[n] += t
        cnt[n] += 1
    print(f"window: launches {win[0][0]}..{win[-1][0]} = step {a.step} ({len(win)} launches, "
          f"serialised cold-cache device time {tot:.1f} ms): compare SHARES")
    print("kernel | launches | share of the step's device time")
    for n, t in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"{n[:50]:50s} {cnt[n]:6d} {100 * t / tot:7.2f}%")
    g = sum(t for n, t in agg.items() if n.startswith("gemm_bf16"))
    print(f"\nGEMM (all gemm_bf16_* launches): {100 * g / tot:.1f}% of the step's device time in the launch list")


if __name__ == "__main__":
    main()
