"""Per-source-line warp-stall samples of one kernel in an ncu report (SASS addresses mapped to
lines with nvdisasm -g on the object file the kernel came from).  Diagnostic tooling.
usage: python scripts/ncu_lines.py REPORT.ncu-rep OBJECT.o MANGLED_SUBSTRING [top]"""
import csv
import re
import subprocess
import sys
import tempfile
import os

rep, obj, key = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
kernels, cur, hdr = [], None, None
for line in src:
    if line.startswith('"Kernel Name"'):
        cur = [line, []]
        kernels.append(cur)
        continue
    if line.startswith('"Address"'):
        hdr = next(csv.reader([line]))
        continue
    if cur is not None:
        cur[1].append(next(csv.reader([line])))
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-gi", os.path.join(d, cub)], capture_output=True, text=True).stdout.split("\n")
funcs = [i for i, l in enumerate(dis) if l.startswith(".text.") and key in l]
print("functions matching:", len(funcs))
for kname, rows in kernels:
    print("==", kname[:160])
    starts = [i for i in funcs]
    # pick the function whose instruction count equals the kernel's row count
    best = None
    for st in starts:
        off2 = {}
        cur_line = None
        for l in dis[st + 1:]:
            if l.startswith(".text."):
                break
            m = re.search(r'//## File "([^"]+)", line (\d+)', l)
            if m:
                cur_line = (m.group(1).split("/")[-1], int(m.group(2)))
                continue
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
            if m:
                off2[int(m.group(1), 16)] = cur_line
        if len(off2) == len(rows):
            best = off2
            break
    if best is None:
        print("  no function with", len(rows), "instructions")
        continue
    base = int(rows[0][0], 16)
    agg, stall = {}, {}
    for r in rows:
        k = best.get(int(r[0], 16) - base)
        s = int(r[2])
        agg[k] = agg.get(k, 0) + s
        for j in range(30, 47):
            if r[j].isdigit() and int(r[j]):
                stall.setdefault(k, {})
                stall[k][hdr[j]] = stall[k].get(hdr[j], 0) + int(r[j])
    tot = sum(agg.values())
    print("  samples", tot)
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        st = sorted(stall.get(k, {}).items(), key=lambda x: -x[1])[:3]
        print("  %6d %5.1f%%  %s  %s" % (v, 100.0 * v / tot, k, ", ".join("%s %d" % (a[6:], b) for a, b in st)))

if len(sys.argv) > 5:          # dump the SASS of one source line with samples: ... LINE
    want = int(sys.argv[5])
    for kname, rows in kernels:
        base = int(rows[0][0], 16)
        for r in rows:
            k = best.get(int(r[0], 16) - base)
            if k and k[1] == want:
                st = sorted(((hdr[j][6:], int(r[j])) for j in range(30, 47) if r[j].isdigit() and int(r[j])), key=lambda x: -x[1])[:2]
                print("%6s  %-60s %s" % (r[2], r[1].strip()[:60], st))
