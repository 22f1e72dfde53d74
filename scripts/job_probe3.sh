mkdir -p gpurun_out
python scripts/chunk_stages.py 65536,131072,200000,400000,1000000 > gpurun_out/chunk_stages.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/launches_65k.csv python scripts/one_proj.py 65536 > /dev/null 2>&1
python -m pytest tests/test_gpu_batch.py -x -q -k cells > gpurun_out/t_cells.txt 2>&1
for g in 8 12 16 24; do MREP_SET_GRID=$g python bench.py --config cfg3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('grid $g', round(d['value']), round(d['ms_per_step'],4), d['config'].get('cell_index'), {k: round(v['ms'],4) for k,v in d['roofline']['stages'].items()}, 'e2e', d['e2e']['value'])" >> gpurun_out/cfg3_grid.txt 2>&1 || tail -5 gpurun_out/ab.log >> gpurun_out/cfg3_grid.txt
done
cat gpurun_out/chunk_stages.txt gpurun_out/t_cells.txt gpurun_out/cfg3_grid.txt
