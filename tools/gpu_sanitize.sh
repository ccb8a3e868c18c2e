# compute-sanitizer passes over every kernel family
mkdir -p gpurun_out; python -m paper_2304_06835_b200._build > gpurun_out/build_san.log 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
