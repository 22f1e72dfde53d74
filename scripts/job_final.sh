mkdir -p gpurun_out
bash scripts/bench_all.sh
TAG=r02 bash scripts/profile_round.sh
for c in cfg2 cfg1 cfg3 cfg4 cfg4q cfg5 cfg6 ref default; do echo "== $c"; cut -c1-300 gpurun_out/bench_$c.json; done
