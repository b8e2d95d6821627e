# compute-sanitizer over every libhgs.so kernel (tools/sanitize_drive.py);
# summaries -> gpurun_out/sanitize_<tool>.txt
set -x
timeout 600 python tools/sanitize_drive.py > gpurun_out/sanitize_plain.txt 2>&1; echo "plain rc=$?"
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no --padding 64"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --kernel-name kns=hgs --print-limit 50 \
    python tools/sanitize_drive.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"
  tail -4 gpurun_out/sanitize_$tool.txt
done
