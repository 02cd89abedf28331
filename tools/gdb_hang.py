# cuda-gdb -batch -p PID -x tools/gdb_hang.py : where is every warp of every
# still-running block of the active kernel (diagnostic for device hangs).
import re
import gdb

gdb.execute("set pagination off")
print(gdb.execute("info cuda kernels", to_string=True))
blocks_txt = gdb.execute("info cuda blocks", to_string=True)
print(blocks_txt)
blocks = []
for m in re.finditer(r"\((\d+),0,0\)\s+\((\d+),0,0\)", blocks_txt):
    blocks += list(range(int(m.group(1)), int(m.group(2)) + 1))
for b in blocks[:8]:
    for t in range(0, 384, 32):
        try:
            gdb.execute(f"cuda block {b} thread {t}", to_string=True)
        except gdb.error:
            continue
        try:
            ln = gdb.execute("info line *$pc", to_string=True).strip()
            ins = gdb.execute("x/1i $pc", to_string=True).strip()
        except gdb.error as e:
            ln, ins = str(e), ""
        print(f"block {b} thread {t}: {ln} | {ins}")
