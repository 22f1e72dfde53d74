# A/B of traversal variants on one config: VARIANTS="A=1,B=2 C=3" CFG=cfg3 bash scripts/ab_cfg3.sh
# (each variant = comma-separated env assignments; MREP_LIB=build/variants/... picks a variant build)
mkdir -p gpurun_out
cfg=${CFG:-cfg3}
out=gpurun_out/ab_$cfg.txt
: > $out
[ -n "$TESTS" ] && python -m pytest $TESTS -x -q 2>&1 | tail -3 >> $out
for v in ${VARIANTS:-MREP_X=0}; do
  envs=$(echo $v | tr ',' ' ')
  env $envs python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['roofline']['stages'].items()})" >> $out 2>&1 || tail -5 gpurun_out/ab.log >> $out
done
