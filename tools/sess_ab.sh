# A/B sweep of the int16x2 kernel shape on config 2 (LOCAL)
rm -f gpurun_out/ab_summary.txt
for cfg in ${AB:-"--i16-rows 16 --force-group 1" "--i16-rows 16 --force-group 2" "--i16-rows 8 --force-group 2" "--i16-rows 8 --force-group 4"}; do
  timeout 300 python bench.py ${cfg//_/ } --e2e-steps 0 --no-cpu-baseline --steps 5 ${BENCH_ARGS} > gpurun_out/ab.log 2>&1
  echo "$cfg :: $(tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['bins'])" 2>&1 | tail -1)" >> gpurun_out/ab_summary.txt
done
cat gpurun_out/ab_summary.txt
