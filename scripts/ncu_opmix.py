"""Instruction mix (warp instructions executed per SASS opcode) of each kernel in an ncu report.
usage: python scripts/ncu_opmix.py REPORT.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
cur, hdr = None, None
kernels = []
for line in src:
    if line.startswith('"Kernel Name"'):
        cur = [line, {}]
        kernels.append(cur)
        continue
    if line.startswith('"Address"'):
        hdr = next(csv.reader([line]))
        continue
    if cur is None or hdr is None:
        continue
    r = next(csv.reader([line]))
    if len(r) < 6:
        continue
    ins = r[hdr.index("Source")].strip()
    toks = ins.split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = ".".join(op.split(".")[:2])
    try:
        cnt = int(r[hdr.index("Instructions Executed")])
    except ValueError:
        continue
    cur[1][op] = cur[1].get(op, 0) + cnt
for name, mix in kernels:
    tot = sum(mix.values())
    print("==", name[15:110], "total warp instructions", tot)
    for op, c in sorted(mix.items(), key=lambda x: -x[1])[:top]:
        print("   %-22s %12d  %5.1f%%" % (op, c, 100.0 * c / max(tot, 1)))
