#!/bin/bash
# Generic GPU session: STEPS env selects what to run (space separated):
#   build tests smoke bench bench_extend bench_cfg3 intpipe ncu_launch ncu_full ncu_pipes
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
STEPS=${STEPS:-"build tests smoke bench"}
python build_native.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
for s in $STEPS; do
  case $s in
    tests) timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log ;;
    smoke) timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log ;;
    bench) timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; tail -3 gpurun_out/bench.log ;;
    bench_extend) timeout 900 python bench.py --mode extend --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_extend.log 2>&1; tail -2 gpurun_out/bench_extend.log ;;
    bench_cfg3) timeout 900 python bench.py --config 3 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS} > gpurun_out/bench_cfg3.log 2>&1; tail -2 gpurun_out/bench_cfg3.log ;;
    bench_cfg4) timeout 900 python bench.py --config 4 --no-cpu-baseline --e2e-steps 1 --steps 3 ${BENCH_ARGS} > gpurun_out/bench_cfg4.log 2>&1; tail -2 gpurun_out/bench_cfg4.log ;;
    bench_cfg5) timeout 900 python bench.py --config 5 --no-cpu-baseline --e2e-steps 1 --steps 3 ${BENCH_ARGS} > gpurun_out/bench_cfg5.log 2>&1; tail -2 gpurun_out/bench_cfg5.log ;;
    intpipe) nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/intpipe tools/intpipe.cu && timeout 120 ./tools/intpipe > gpurun_out/intpipe.jsonl 2>&1 ;;
    ncu_launch) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_launch.log 2>&1 ;;
    ncu_full) timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:${NCU_KERNEL:-dp_i16_kernelILi1ELi16E}" -s ${NCU_SKIP:-1} -c ${NCU_COUNT:-1} -o gpurun_out/prof_${NCU_TAG:-dp} -f python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --pairs ${NCU_PAIRS:-300000} ${BENCH_ARGS} > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log ;;
    ncu_pipes) timeout 600 ncu --clock-control none --metrics sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmalite.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg,smsp__inst_executed.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__inst_executed_pipe_uniform.sum,gpc__cycles_elapsed.avg.per_second --csv --log-file gpurun_out/intpipe_ncu.csv ./tools/intpipe > /dev/null 2>&1 ;;
    *) eval "$s" ;;
  esac
done
echo done
