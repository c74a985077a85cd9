# compute-sanitizer over one pass of every kernel family (scripts/sanitize_run.py); summaries -> gpurun_out
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python scripts/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1; tail -1 gpurun_out/sanitize_plain.log
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(tail -2 gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
