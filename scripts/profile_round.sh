# launch lists of bench.py's timed steps (NVTX range bench_timed) per config,
# gpu__time_duration.sum per launch (cold, serialised: shares, not absolutes)
mkdir -p gpurun_out
for c in cfg2 cfg3 cfg4 cfg5; do
  n=""; [ $c = cfg5 ] && n="--n 4000000"
  ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_timed/" \
      --csv --log-file gpurun_out/launches_$c.csv \
      python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline $n > gpurun_out/ll_$c.log 2>&1
done
