mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest -q -x tests/test_gpu_banded_i16.py tests/test_gpu_banded.py > gpurun_out/pt_band.log 2>&1; tail -3 gpurun_out/pt_band.log
python tools/probe_band_bins.py 2 1000000 0
python tools/probe_band_bins.py 4 100000 0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dp_g1 -s 2 -c 1 -o gpurun_out/prof_band2 -f python tools/probe_band_bins.py 2 1000000 0 > gpurun_out/ncu_band.log 2>&1
tail -1 gpurun_out/ncu_band.log
