# End-of-round-2 evidence: GPU tests, smoke, bench lines for every config, the reference arm, the
# ncu launch list of the default bench command, and one ncu --set full capture of dp_g1_kernel.
# Outputs under gpurun_out/final2/ (copied to profiles/r02_final/ afterwards).
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/final2; mkdir -p $O
python build_native.py > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 300 $O/bench_default.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>&1
for a in "--mode extend" "--config 3" "--config 4 --steps 3" "--config 5 --steps 3" "--config 5 --steps 3 --grouped" "--config 1" "--p-n 0.001" "--config 4 --steps 2 --band 100" "--band 100" "--config 4 --pairs 4000 --steps 3" "--config 5 --pairs 1250000 --steps 3"; do
  n=$(echo "$a" | tr -d ' -' ); timeout 900 python bench.py $a --no-cpu-baseline --e2e-steps 1 > $O/bench_$n.json 2> $O/bench_$n.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_config2.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --start-steps 0 --ksw-steps 0 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_list.py $O/launches_config2.csv > $O/launches_config2_summary.txt 2>&1; head -8 $O/launches_config2_summary.txt
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:dp_g1_kernelILi0ELi4ELb0ELb0E" -s 1 -c 1 -o $O/prof_g1_final -f python bench.py --steps 1 --warmup 1 --e2e-steps 0 --start-steps 0 --ksw-steps 0 --no-cpu-baseline > $O/ncu_full.log 2>&1; tail -2 $O/ncu_full.log
echo done
