# register-cap A/B (base vs build/variants v1, v2), e2e timeline, approx-handle leak probe
mkdir -p gpurun_out
for cfg in cfg2 cfg3 cfg6; do
  VARIANTS="MREP_X=0 MREP_LIB=build/variants/libmrep_v1.so MREP_LIB=build/variants/libmrep_v2.so" CFG=$cfg bash scripts/ab_cfg3.sh
done
for v in "" build/variants/libmrep_v1.so build/variants/libmrep_v2.so; do
  env ${v:+MREP_LIB=$v} python bench.py --config cfg5 --n 20000000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 $v', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['roofline']['stages'].items()})" >> gpurun_out/ab_cfg5.txt 2>&1
done
python scripts/e2e_trace.py cfg2 4 > gpurun_out/e2e_trace.txt 2>&1
compute-sanitizer --tool memcheck --leak-check full python scripts/leak_probe.py > gpurun_out/leak_probe.txt 2>&1
cat gpurun_out/ab_*.txt
