mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 -k "not c3_full and not pcg_parity_c5[None]" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 600 python bench.py --config c1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; echo b1=$?
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo b3=$?
tail -3 gpurun_out/*.log
