mkdir -p gpurun_out
for c in ${CONFIGS:-c1 c2 c4 c5}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg_$c.json 2>> gpurun_out/bench_cfg.err; echo bench_$c=$?
  python -c "
import json; d=json.load(open('gpurun_out/bench_cfg_$c.json')); print('$c value %.3e ms %.3f frac %.3f launches %d'%(d['value'],d['ms_per_step'],d['roofline']['frac'] or 0, d['gpu_launches'])); print({k:v['ms_per_step'] for k,v in list(d['kernels'].items())[:10]})"
done
