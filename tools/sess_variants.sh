# A/B of library variants built by tools/variants.py (VARIANTS="base name1=-DX ..."), bench args in BENCH_ARGS
rm -f gpurun_out/var_summary.txt
VARIANTS_PREBUILT=1 python tools/variants.py ${VARIANTS} > gpurun_out/variants_build.log 2>&1 || { tail -30 gpurun_out/variants_build.log; exit 1; }
for rep in 1 ${REPS:-}; do
for v in ${VARIANTS}; do
  name=${v%%=*}
  SALOBA_LIB=build/variants/$name/libsaloba.so timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --steps 5 ${BENCH_ARGS} > gpurun_out/var_$name.log 2>&1
  echo "$name :: $(tail -1 gpurun_out/var_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])" 2>&1 | tail -1)" >> gpurun_out/var_summary.txt
done
done
cat gpurun_out/var_summary.txt
