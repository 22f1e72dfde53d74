mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/ab_emit.txt
for c in cfg2 cfg3 cfg6 cfg1; do
  MREP_SET_GRID=0 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['roofline']['stages'].items()}, 'e2e', round(d['e2e']['value']))" >> gpurun_out/ab_emit.txt 2>&1 || tail -3 gpurun_out/ab.log >> gpurun_out/ab_emit.txt
done
python bench.py --config cfg5 --n 20000000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1
tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 2e7', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['roofline']['stages'].items()})" >> gpurun_out/ab_emit.txt 2>&1
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:wave_emit \
    -o gpurun_out/r02_cfg2_emit -f python scripts/one_proj.py 1000000 > gpurun_out/ncu_emit.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/ab_emit.txt
