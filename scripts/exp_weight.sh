for v in mid next; do echo "== weight $v"; PMG_EXPERIMENT_WEIGHT=$v timeout 600 python scripts/table1_sweep.py exp 3,4,5,9,13 2>&1 | grep row; done
for sc in 1.5 2.0; do echo "== weight scale $sc"; PMG_EXPERIMENT_WEIGHT=scale PMG_EXPERIMENT_SCALE=$sc timeout 600 python scripts/table1_sweep.py exp 3,5,9,13 2>&1 | grep row; done
