# Round-2 A/B session: parity subset, then bench lines for library variants (VARIANTS="name=flags ..."; the
# in-tree build is "base"), then optionally an ncu capture of one kernel (NCU_KERNEL regex).
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -n "${TESTS}" ]; then
  timeout 1500 python -m pytest ${TESTS} -x -q > gpurun_out/pytest_ab.log 2>&1; tail -3 gpurun_out/pytest_ab.log
fi
VARIANTS_PREBUILT=1 python tools/variants.py ${VARIANTS} > gpurun_out/variants_build.log 2>&1
rm -f gpurun_out/ab_summary.txt
for args in "${BENCH_SETS[@]:-}"; do :; done
IFS=';' read -ra SETS <<< "${BENCHES:---config 2}"
for rep in 1 ${REPS:-}; do
for b in "${SETS[@]}"; do
for v in base ${VARIANTS}; do
  name=${v%%=*}
  lib=paper_2301_09310_b200/libsaloba.so; [ "$name" != base ] && lib=build/variants/$name/libsaloba.so
  SALOBA_LIB=$lib timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline --start-steps 0 --ksw-steps 0 --no-graph --steps 5 $b > gpurun_out/ab_run.log 2>&1
  echo "$name [$b] :: $(tail -1 gpurun_out/ab_run.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['achieved'], r['frac'], r['bins'])" 2>&1 | tail -1)" >> gpurun_out/ab_summary.txt
done; done; done
cat gpurun_out/ab_summary.txt
if [ -n "${NCU_KERNEL}" ]; then
  timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:${NCU_KERNEL}" -s ${NCU_SKIP:-1} -c 1 -o gpurun_out/prof_${NCU_TAG:-ab} -f python bench.py --steps 1 --warmup 1 --e2e-steps 0 --start-steps 0 --ksw-steps 0 --no-graph --no-cpu-baseline ${NCU_ARGS:---pairs 300000} > gpurun_out/ncu_ab.log 2>&1; tail -2 gpurun_out/ncu_ab.log
fi
echo done
