# bench every config once (LOCAL) + config 2 EXTEND
rm -f gpurun_out/configs_summary.txt
for a in "--config 2 --mode extend" "--config 3" "--config 4 --steps 2" "--config 5 --steps 2" "--config 5 --steps 2 --grouped" "--config 1"; do
  timeout 600 python bench.py $a --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS} > gpurun_out/cfg.log 2>&1
  echo "$a :: $(tail -1 gpurun_out/cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['bins'], d['e2e']['value'])" 2>&1 | tail -1)" >> gpurun_out/configs_summary.txt
done
cat gpurun_out/configs_summary.txt
