# compute-sanitizer evidence: memcheck, racecheck (shared memory), synccheck over a small
# workload that launches every kernel (tools/sanitize_run.py).  Summaries -> gpurun_out/sanitizer_*.txt
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python tools/sanitize_run.py > gpurun_out/sanitizer_plain.txt 2>&1; tail -3 gpurun_out/sanitizer_plain.txt
for tool in memcheck racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitizer_$tool.txt
done
echo done
