# per-bin block shares on/off (SALOBA_BIN_SHARES=0) on the skewed configs
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/shares_summary.txt
for a in ${SHARE_CFGS:-"--config_5_--pairs_1250000_--steps_3" "--config_4_--pairs_4000_--steps_3" "--config_3_--steps_5" "--config_5_--steps_2" "--steps_5"}; do
  for sh in 1 0; do
    SALOBA_BIN_SHARES=$sh timeout ${BT:-300} python bench.py ${a//_/ } --e2e-steps 0 --no-cpu-baseline --start-steps 0 --ksw-steps 0 > gpurun_out/shares.log 2>&1
    echo "$a shares=$sh :: $(tail -1 gpurun_out/shares.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['achieved'], r['frac'], r['bins'])" 2>&1 | tail -1)" >> gpurun_out/shares_summary.txt
  done
done
cat gpurun_out/shares_summary.txt
