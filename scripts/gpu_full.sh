# Full GPU session: parity suite, default bench (c3 + cpu baseline), other configs,
# ncu launch list + full capture of the top-level Schwarz kernel.
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=10 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_rc=$?
for c in c1 c2 c4 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2>> gpurun_out/bench_$TAG.err; echo bench_$c=$?
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_reference.json 2>> gpurun_out/bench_$TAG.err; echo ref=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fdm_eoc|k_apply_mma|k_fold2" -c 3 -o gpurun_out/prof_full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu_full=$?
