# every bench line of the round into gpurun_out/bench_<cfg>.json (+ logs)
mkdir -p gpurun_out
for c in cfg2 cfg1 cfg3 cfg4 cfg4q cfg6; do
  timeout 600 python bench.py --config $c --steps 50 --warmup 5 > gpurun_out/bench_$c.log 2>&1
  tail -1 gpurun_out/bench_$c.log > gpurun_out/bench_$c.json
done
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 > gpurun_out/bench_cfg5.log 2>&1
tail -1 gpurun_out/bench_cfg5.log > gpurun_out/bench_cfg5.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref.json
python bench.py > gpurun_out/bench_default.log 2>&1
tail -1 gpurun_out/bench_default.log > gpurun_out/bench_default.json
