#!/bin/bash
# First GPU session: build, int-pipe microbench, GPU tests, smoke, bench, ncu launch list.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
python build_native.py > gpurun_out/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/intpipe tools/intpipe.cu && timeout 120 ./tools/intpipe > gpurun_out/intpipe.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --pairs 200000 > gpurun_out/ncu_launch_bench.log 2>&1
echo done
