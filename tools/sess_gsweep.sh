for g in 1 2 8; do timeout 300 python bench.py --force-group $g --e2e-steps 0 --no-cpu-baseline --steps 5 > gpurun_out/bench_g$g.log 2>&1; done
