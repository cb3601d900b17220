set -x
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest -q -x tests/test_gpu_banded_i16.py tests/test_gpu_banded.py tests/test_gpu_parity.py tests/test_gpu_counters.py tests/test_gpu_traceback.py > gpurun_out/pt1.log 2>&1
tail -5 gpurun_out/pt1.log
timeout 300 python bench.py > gpurun_out/b_default.json 2> gpurun_out/b_default.err; cat gpurun_out/b_default.json
timeout 300 python bench.py --config 2 > gpurun_out/b_c2.json 2>&1; tail -1 gpurun_out/b_c2.json
timeout 300 python bench.py --config 2 --band 100 > gpurun_out/b_c2b.json 2>&1; tail -1 gpurun_out/b_c2b.json
timeout 300 python bench.py --config 4 --band 100 > gpurun_out/b_c4b.json 2>&1; tail -1 gpurun_out/b_c4b.json
