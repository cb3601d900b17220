# Variant A/B session: VARIANTS="name ..." (built here by tools/variants.py under build/variants/<name>),
# each timed with bench.py ${VARGS}; summary line per variant in gpurun_out/var_summary.txt.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
rm -f gpurun_out/var_summary.txt
for v in ${VARIANTS}; do
  for args in "${VARGS:---e2e-steps 0 --no-cpu-baseline --start-steps 0 --ksw-steps 0 --steps 10}"; do
    lib=build/variants/$v/libsaloba.so; [ "$v" = main ] && lib=paper_2301_09310_b200/libsaloba.so
    SALOBA_LIB=$lib timeout 600 python bench.py $args > gpurun_out/var_$v.log 2>&1
    echo "$v [$args] :: $(tail -1 gpurun_out/var_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['achieved'], r['frac'], r['bins'], d['clocks'])" 2>&1 | tail -1)" >> gpurun_out/var_summary.txt
  done
done
cat gpurun_out/var_summary.txt
