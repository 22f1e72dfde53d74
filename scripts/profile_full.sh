# ncu --set full of ONE projection call per config (the "timed" NVTX range of
# scripts/one_*.py), exported .ncu-rep into gpurun_out/ for ncu_summarize.py
mkdir -p gpurun_out
tag=${TAG:-r02}
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
    -o gpurun_out/${tag}_cfg2_full -f python scripts/one_proj.py 1000000 > gpurun_out/${tag}_ncu_cfg2.log 2>&1
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
    -o gpurun_out/${tag}_cfg3_full -f python scripts/one_batch.py > gpurun_out/${tag}_ncu_cfg3.log 2>&1
