"""Warp-stall samples of one kernel in an ncu report, attributed to source lines.

    python tools/ncu_lines.py REPORT.ncu-rep attn_bwd_fused_sm100 [--top 30]

ncu's csv source page lists stall samples per SASS address; the line table comes
from the cubin embedded in libstp.so (built with -lineinfo; the report must come
from the same build).  Prints the share of all samples per (file, line) with the
three largest stall reasons.
"""
import argparse
import collections
import csv
import os
import re
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2510_27257_b200", "libstp.so")


def line_table(kernel):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=d, check=True, capture_output=True)
        for f in sorted(os.listdir(d)):
            dis = subprocess.run(["nvdisasm", "--print-line-info", "-c", os.path.join(d, f)], capture_output=True,
                                 text=True).stdout
            hdr = re.search(r"^\.text\.(\S*%s\S*):" % re.escape(kernel), dis, re.M)
            if hdr:
                break
        else:
            raise SystemExit(f"{kernel} not found in {LIB}")
    body = dis[hdr.end():]
    nxt = re.search(r"^\s*\.section\s", body, re.M)
    body = body[:nxt.start()] if nxt else body
    table, cur = {}, None
    for ln in body.split("\n"):
        m = re.search(r'"([^"]+)", line (\d+)', ln)
        if "//## File" in ln and m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
        a = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if a and cur:
            table.setdefault(int(a.group(1), 16), cur)
    return table


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))[1:]
    hdr, data = rows[0], rows[1:]
    i_all = hdr.index("Warp Stall Sampling (All Samples)")
    reasons = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    table = line_table(a.kernel)
    base = int(data[0][0], 16)
    tot = 0.0
    agg = collections.defaultdict(float)
    why = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in data:
        k = table.get(int(r[0], 16) - base, ("?", 0))
        v = float(r[i_all] or 0)
        tot += v
        agg[k] += v
        for i, nm in reasons:
            why[k][nm] += float(r[i] or 0)
    src = {}
    for k, v in sorted(agg.items(), key=lambda t: -t[1])[:a.top]:
        path = os.path.join(ROOT, "paper_2510_27257_b200", "csrc", k[0])
        if k[0] not in src:
            src[k[0]] = open(path).read().split("\n") if os.path.exists(path) else []
        text = src[k[0]][k[1] - 1].strip()[:64] if 0 < k[1] <= len(src[k[0]]) else ""
        top = sorted(why[k].items(), key=lambda t: -t[1])[:3]
        print(f"{100 * v / tot:5.1f}%  {k[0]}:{k[1]:<5} {text:64s} "
              + ", ".join(f"{n} {100 * x / tot:.1f}" for n, x in top))


if __name__ == "__main__":
    main()
