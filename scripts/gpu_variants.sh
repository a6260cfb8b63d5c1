# Diagnostic A/B: c3 bench with the in-tree library and each variants/lib_*.so (PMG_LIB), plus the
# FDM phase probe.  Variants are -D builds of the same sources (paper_1612_04796_b200/build.py --out).
mkdir -p gpurun_out
TAG=${TAG:-v}
CFG=${CFG:-c3}
timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/var_${TAG}_main.json 2> gpurun_out/var_${TAG}_main.err; echo main=$?
for v in ${VARIANTS:-}; do
  PMG_LIB=variants/lib_$v.so timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/var_${TAG}_$v.json 2> gpurun_out/var_${TAG}_$v.err; echo $v=$?
done
if [ -f variants/lib_phase.so ] && [ -n "$PHASE" ]; then
  PMG_LIB=variants/lib_phase.so timeout 300 python scripts/phase_probe.py $CFG > gpurun_out/phase_${TAG}.log 2>&1; echo phase=$?
fi
python - <<'PY'
import json, glob, os
tag = os.environ.get("TAG", "v")
for f in sorted(glob.glob(f"gpurun_out/var_{tag}_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k = d.get("kernels", {})
    print(os.path.basename(f), "ms/step %.4f" % d["ms_per_step"],
          " ".join("%s=%.4f" % (n, k[n]["ms_per_cycle"]) for n in list(k)[:8]))
PY
