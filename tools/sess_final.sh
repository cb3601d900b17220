# End-of-round evidence session: tests, bench lines for every config, reference arm, ncu launch
# list and traffic of the bench command.  Outputs under gpurun_out/final/.
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
python build_native.py > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 300 $O/bench_default.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2>&1
for a in "--mode extend" "--config 3" "--config 4 --steps 3" "--config 5 --steps 3" "--config 5 --steps 3 --grouped" "--config 1" "--p-n 0.001" "--config 4 --steps 2 --band 100"; do
  n=$(echo "$a" | tr -d ' -' ); timeout 900 python bench.py $a --no-cpu-baseline --e2e-steps 1 > $O/bench_$n.json 2> $O/bench_$n.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_config2.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --start-steps 0 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_list.py $O/launches_config2.csv > $O/launches_config2_summary.txt 2>&1; head -8 $O/launches_config2_summary.txt
echo done
