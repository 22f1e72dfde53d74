mkdir -p gpurun_out
: > gpurun_out/ab_cfg3_stage.txt
for v in "MREP_X=0" "MREP_STAGE=1" "MREP_STAGE=1,MREP_STAGE_CTAS=2" "MREP_SET_GRID=12" "MREP_SET_GRID=10"; do
  envs=$(echo $v | tr ',' ' ')
  env MREP_SET_GRID=0 $envs python bench.py --config cfg3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],4), d['config'].get('cell_index'), {k: round(v['ms'],4) for k,v in d['roofline']['stages'].items()}, 'e2e', round(d['e2e']['value']))" >> gpurun_out/ab_cfg3_stage.txt 2>&1 || tail -3 gpurun_out/ab.log >> gpurun_out/ab_cfg3_stage.txt
done
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/launches_prep_cfg3.csv python scripts/one_prep.py cfg3 > gpurun_out/ncu_prep.log 2>&1
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:approx_eval -c 3 \
    -o gpurun_out/r02_prep_full -f python scripts/one_prep.py cfg3 > gpurun_out/ncu_prep_full.log 2>&1
MREP_SET_GRID=0 python bench.py --config cfg2 --steps 30 --warmup 5 > gpurun_out/bench_cfg2_prep.log 2>&1
MREP_SET_GRID=0 python bench.py --config cfg3 --steps 30 --warmup 5 > gpurun_out/bench_cfg3_prep.log 2>&1
cat gpurun_out/ab_cfg3_stage.txt; tail -c 1500 gpurun_out/bench_cfg3_prep.log
