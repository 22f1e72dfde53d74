mkdir -p gpurun_out
: > gpurun_out/dmma_ab.txt
for c in cfg2 cfg6; do
  python scripts/dmma_check.py $c /tmp/a_$c.npz > /dev/null 2>&1
  MREP_TRAV_DMMA=1 python scripts/dmma_check.py $c /tmp/b_$c.npz > /dev/null 2>&1
  echo "== $c" >> gpurun_out/dmma_ab.txt; python scripts/dmma_check.py cmp /tmp/a_$c.npz /tmp/b_$c.npz >> gpurun_out/dmma_ab.txt 2>&1
done
python scripts/dmma_check.py cfg5 /tmp/a_cfg5.npz 4000000 > /dev/null 2>&1
MREP_TRAV_DMMA=1 python scripts/dmma_check.py cfg5 /tmp/b_cfg5.npz 4000000 > /dev/null 2>&1
echo "== cfg5 (4e6)" >> gpurun_out/dmma_ab.txt; python scripts/dmma_check.py cmp /tmp/a_cfg5.npz /tmp/b_cfg5.npz >> gpurun_out/dmma_ab.txt 2>&1
for v in "MREP_X=0" "MREP_TRAV_DMMA=1"; do
  for c in cfg2 cfg6; do
    env $v python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab.log 2>&1
    tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['roofline']['stages'].items()}, d['roofline']['per_query'])" >> gpurun_out/dmma_ab.txt 2>&1
  done
  env $v python bench.py --config cfg5 --n 20000000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg5', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['roofline']['stages'].items()}, d['roofline']['per_query'])" >> gpurun_out/dmma_ab.txt 2>&1
done
MREP_TRAV_DMMA=1 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:wave_traverse_dmma -o gpurun_out/r02_trav_dmma -f python scripts/one_proj.py 1000000 > gpurun_out/ncu_dmma.log 2>&1
cat gpurun_out/dmma_ab.txt
