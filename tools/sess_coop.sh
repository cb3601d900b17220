# long-pair batches with and without the cooperative kernel (SALOBA_COOP_PAIRS=0 disables it)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/coop_summary.txt
for a in ${COOP_CFGS:-"--config_5_--pairs_1250000_--steps_3" "--config_4_--pairs_4000_--steps_3" "--config_4_--pairs_12500_--steps_3"} ${COOP_EXTRA}; do
  for cp in default 0; do
    if [ $cp = default ]; then unset SALOBA_COOP_PAIRS; else export SALOBA_COOP_PAIRS=$cp; fi
    timeout ${BT:-600} python bench.py ${a//_/ } --e2e-steps 0 --no-cpu-baseline --start-steps 0 --ksw-steps 0 > gpurun_out/coop.log 2>&1
    echo "$a coop_pairs=$cp :: $(tail -1 gpurun_out/coop.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['achieved'], r['frac'], r['bins'])" 2>&1 | tail -1)" >> gpurun_out/coop_summary.txt
  done
done
unset SALOBA_COOP_PAIRS
cat gpurun_out/coop_summary.txt
