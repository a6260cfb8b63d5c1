# A/B timing in one GPU session: bench runs given as "label|args|lib" triples in $RUNS (';'-separated)
mkdir -p gpurun_out
TAG=${TAG:-ab}
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -k "$TESTS" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest_rc=$?
  tail -4 gpurun_out/pytest_$TAG.log
fi
IFS=';' read -ra R <<< "$RUNS"
for spec in "${R[@]}"; do
  IFS='|' read -r label bargs lib <<< "$spec"
  if [ -n "$lib" ]; then export PMG_LIB=$lib; else unset PMG_LIB; fi
  timeout 600 python bench.py --no-cpu-baseline $bargs > gpurun_out/ab_${TAG}_$label.json 2> gpurun_out/ab_${TAG}_$label.err; echo $label=$?
done
unset PMG_LIB
python - <<'PY'
import json, glob, os
tag = os.environ.get("TAG", "ab")
for f in sorted(glob.glob(f"gpurun_out/ab_{tag}_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k = d.get("kernels", {})
    print(os.path.basename(f), "ms/step %.4f val %.3e" % (d["ms_per_step"], d["value"]), "clk", d["clocks"].get("sm_mhz"),
          " ".join("%s=%.4f" % (n, k[n]["ms_per_cycle"]) for n in list(k)[:9]))
PY
