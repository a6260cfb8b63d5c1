mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -k "${K:-smoother or vcycle_parity or edge or rate}" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-cpu-baseline ${BARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('value %.3e ms %.3f'%(d['value'],d['ms_per_step']), d['roofline']); print({k:v['ms_per_step'] for k,v in list(d['kernels'].items())[:8]})"
