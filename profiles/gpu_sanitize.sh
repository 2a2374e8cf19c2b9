# compute-sanitizer over every hot-path kernel (small shapes); logs in gpurun_out/
TAG="${1:-r02}"
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python profiles/sanitize_driver.py > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize driver done' gpurun_out/sanitize_${tool}_$TAG.log | tr '\n' ' ')"
done
