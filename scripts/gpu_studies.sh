mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=8 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python scripts/table1_sweep.py $TAG > gpurun_out/table1_$TAG.txt 2>&1; echo table1=$?
timeout 1500 python scripts/aniso_study.py $TAG > gpurun_out/aniso_$TAG.txt 2>&1; echo aniso=$?
tail -60 gpurun_out/aniso_$TAG.txt
