mkdir -p gpurun_out
TAG=${TAG:-n}
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline ${BARGS}"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_fdm_mma|k_apply_mma|k_fold}" -c ${NCOUNT:-3} -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_$TAG.log
