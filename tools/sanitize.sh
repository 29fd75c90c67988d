# compute-sanitizer over a small pass of the hot path (SURVEY §5 race/memory checks); summaries
# to gpurun_out/sanitize_<tool>.txt.  Usage: bash tools/sanitize.sh
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_case.py \
      > gpurun_out/sanitize_$t.txt 2>&1
  echo "$t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|error' gpurun_out/sanitize_$t.txt | tail -2 | tr '\n' ' ')"
done
