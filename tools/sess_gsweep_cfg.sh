rm -f gpurun_out/gsweep.txt
for c in ${CFGS:-5 3 4}; do for g in ${GS:-1 2 4 8 16}; do
  st=5; [ $c -ge 4 ] && st=2
  timeout 400 python bench.py --config $c --force-group $g --e2e-steps 0 --no-cpu-baseline --steps $st --pairs ${PAIRS:-200000} > gpurun_out/gs.log 2>&1
  echo "cfg $c G $g :: $(tail -1 gpurun_out/gs.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['bins'])" 2>&1 | tail -1)" >> gpurun_out/gsweep.txt
done; done
cat gpurun_out/gsweep.txt
