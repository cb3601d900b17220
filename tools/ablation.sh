#!/bin/bash
# On-B200 ablation of the design choices (§V-C "ablation", P:1269-1296;
# Table I "tab:moti" traffic).  Run on the GPU box:
#   gpurun -- 'bash tools/ablation.sh'   -> gpurun_out/ablation/*.{log,csv}; summarise with
#   python tools/ablation_summary.py     -> profiles/r01_ablation.json
# Sweeps (each a bench.py run, DP kernels timed by CUDA events on the launching stream):
#   * subwarp size G in {1,2,4,8,16,32} (force_group), int16x2 path, configs 2 and 4;
#   * the same on the exact int32 path (force_path=1) = the paper's scalar-int32 kernel shape;
#   * scheduler off (keep_order=1: no length sort) on config 3 and config 5 (skewed lengths);
# and, per G on config 2, one ncu pass of traffic / pipe counters for the DP kernel.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ablation
python build_native.py > gpurun_out/ablation/build.log 2>&1 || { tail -30 gpurun_out/ablation/build.log; exit 1; }
B="python bench.py --no-cpu-baseline --e2e-steps 0 --start-steps 0 --no-graph"
for g in 1 2 4 8 16 32; do
  timeout 300 $B --config 2 --pairs 300000 --steps 5 --force-group $g > gpurun_out/ablation/c2_i16_g$g.log 2>&1
  timeout 300 $B --config 2 --pairs 300000 --steps 3 --force-group $g --force-path 1 > gpurun_out/ablation/c2_i32_g$g.log 2>&1
  timeout 300 $B --config 4 --pairs 4000 --steps 2 --force-group $g > gpurun_out/ablation/c4_i16_g$g.log 2>&1
done
for c in 3 5; do
  timeout 300 $B --config $c --pairs 300000 --steps 3 > gpurun_out/ablation/c${c}_sched.log 2>&1
  timeout 300 $B --config $c --pairs 300000 --steps 3 --keep-order 1 > gpurun_out/ablation/c${c}_nosched.log 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__inst_executed_pipe_alu.sum,smsp__inst_executed.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for g in 1 2 4 8 16 32; do
  timeout 600 ncu --clock-control none --metrics $M -k regex:dp_i16_kernel --csv --log-file gpurun_out/ablation/ncu_c2_g$g.csv \
    $B --config 2 --pairs 100000 --steps 1 --warmup 1 --force-group $g > /dev/null 2>&1
done
echo done
