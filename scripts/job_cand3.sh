mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_project.py -x -q -k "cand" > gpurun_out/t_cand.txt 2>&1; echo rc=$? >> gpurun_out/t_cand.txt
python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_cand.log 2>&1
tail -1 gpurun_out/b_cand.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['e2e_reference_cand']['value'], json.dumps(d['roofline']['cand_exact']))" > gpurun_out/cand_stage.txt 2>&1
EXTRA_FLAGS=1536 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_cand.csv python scripts/one_proj.py 1000000 > /dev/null 2>&1
tail -3 gpurun_out/t_cand.txt; cat gpurun_out/cand_stage.txt; grep -i "cand" gpurun_out/launches_cand.csv | awk -F'","' '{print $5, $NF}' | head
