mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
export SANITIZE_N=1024
bash scripts/sanitize_all.sh
MREP_TRAV_DMMA=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py curve > gpurun_out/sanitizer/memcheck_dmma.log 2>&1; echo "exit=$?" >> gpurun_out/sanitizer/memcheck_dmma.log
MREP_TRAV_DMMA=1 timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py curve > gpurun_out/sanitizer/racecheck_dmma.log 2>&1; echo "exit=$?" >> gpurun_out/sanitizer/racecheck_dmma.log
tail -3 gpurun_out/pytest_gpu.log; grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|LEAK SUMMARY\|exit=" gpurun_out/sanitizer/*.log
