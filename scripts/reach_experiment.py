"""Reading-R6 experiment: Table 1 rows 1, 2, 7, 8 (FixedNodes(1)) at
P = 4, 8, 16, 32 with the library given by PMG_LIB; prints -lg rho next to the paper's values."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.table1_sweep import PAPER, run_case

rows = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "7", "8"])]
out = {}
for row in rows:
    basis, solver, ov, paper = PAPER[row]
    for P, want in zip([4, 8, 16, 32], paper):
        r = run_case(basis, solver, ov, P, 128 // P)
        out["%d/%d" % (row, P)] = {"lg": r["lg"], "paper": want, "n_o": r["n_o"]}
        print("row %2d P=%2d  -lg rho %.3f  paper %.2f  diff %+.3f" % (row, P, r["lg"], want, r["lg"] - want), flush=True)
print(json.dumps(out))
