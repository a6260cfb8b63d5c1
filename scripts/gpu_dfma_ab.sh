# DMMA vs DFMA A/B at n = 3, 5, 9 (north_star: DMMA only where the batched mode product is a real
# dense contraction, justified by ncu counters).  variants/lib_dfma.so = -DPMG_FORCE_DFMA build:
# levels with n <= 9 run the scalar FP64-FMA kernels k_fdm / k_apply instead of the DMMA line GEMMs.
mkdir -p gpurun_out
TAG=${TAG:-dfma}
TAG=$TAG RUNS="c3_dmma|--steps 20 --no-sub-configs|;c3_dfma|--steps 20 --no-sub-configs|variants/lib_dfma.so;c2_dmma|--config c2 --steps 20|;c2_dfma|--config c2 --steps 20|variants/lib_dfma.so;c1_dmma|--config c1 --steps 50|;c1_dfma|--config c1 --steps 50|variants/lib_dfma.so" bash scripts/gpu_ab.sh
python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain_${TAG}.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"k_fdm|k_apply" -c 12 -o gpurun_out/prof_${TAG}_dmma python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_${TAG}_a.log 2>&1; echo ncu_a=$?
PMG_LIB=variants/lib_dfma.so python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain_${TAG}_b.log 2>&1 && \
PMG_LIB=variants/lib_dfma.so timeout 900 ncu --set full --clock-control none -k regex:"k_fdm|k_apply" -c 12 -o gpurun_out/prof_${TAG}_dfma python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_${TAG}_b.log 2>&1; echo ncu_b=$?
