# compute-sanitizer over every device path (scripts/sanitize.py), one log per tool
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python scripts/sanitize.py > gpurun_out/sanitizer/$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/sanitizer/$tool.log
done
