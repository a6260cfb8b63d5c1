mkdir -p gpurun_out
timeout ${T:-2400} python -m pytest tests -m gpu -q --timeout 900 --durations=15 ${ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -40 gpurun_out/pytest_gpu.log
