mkdir -p gpurun_out
EXTRA_FLAGS=1536 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:cand_ -o gpurun_out/r02_candcells_full -f python scripts/one_proj.py 1000000 > gpurun_out/ncu_candcells.log 2>&1
python bench.py --config cfg2 --steps 30 --warmup 5 > gpurun_out/bench_cfg2.log 2>&1
tail -1 gpurun_out/bench_cfg2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], json.dumps(d['e2e_reference_cand']), json.dumps(d['roofline']['cand_exact']), d.get('preparation',{}).get('cubics_per_s'))"
