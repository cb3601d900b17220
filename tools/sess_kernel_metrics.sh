# Per-kernel pipe / issue / DRAM metrics of every kernel family (ncu --metrics, one pass each).
cd $GRAFT_REPO_ROOT
O=gpurun_out/kmetrics; mkdir -p $O
python build_native.py > $O/build.log 2>&1
M=gpu__time_duration.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
run() { name=$1; shift; timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/$name.csv $B "$@" > /dev/null 2>&1; echo "$name done"; }
run default --start-steps 1
run queryN --p-n 0.01 --start-steps 0
run int32_g2 --pairs 300000 --force-path 1 --force-group 2 --start-steps 0
run extend --mode extend --start-steps 0
run banded_c4 --config 4 --pairs 20000 --band 100 --start-steps 0
run long_c4 --config 4 --pairs 20000 --start-steps 0
