export SANITIZE_N=1024
bash scripts/sanitize_all.sh
bash scripts/profile_full.sh
bash scripts/profile_round.sh
grep -h "exit=" gpurun_out/sanitizer/*.log; grep -h "ERROR SUMMARY" gpurun_out/sanitizer/*.log
ls -la gpurun_out
