# One GPU session: parity tests, bench (c3 default + other configs), ncu launch list + full capture.
mkdir -p gpurun_out
TAG=${TAG:-r1}
if [ -z "$SKIP_TESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=10 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu_$TAG.log
fi
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_rc=$?
for c in ${CONFIGS:-c1 c2 c4 c5}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2>> gpurun_out/bench_$TAG.err; echo bench_$c=$?
done
if [ -z "$SKIP_NCU" ]; then
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fdm -s 2 -c 2 -o gpurun_out/prof_fdm_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu_full=$?
fi
ls -la gpurun_out
