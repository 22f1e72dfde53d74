mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_project.py tests/test_gpu_batch.py tests/test_gpu_api.py tests/test_gpu_nearest.py -x -q > gpurun_out/t_clip.txt 2>&1; echo rc=$? >> gpurun_out/t_clip.txt
: > gpurun_out/ab_clip.txt
for c in cfg2 cfg3 cfg6 cfg1; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['roofline']['stages'].items()}, 'e2e', round(d['e2e']['value']))" >> gpurun_out/ab_clip.txt 2>&1
done
python bench.py --config cfg5 --n 20000000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1
tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['roofline']['stages'].items()})" >> gpurun_out/ab_clip.txt 2>&1
tail -3 gpurun_out/t_clip.txt; cat gpurun_out/ab_clip.txt
