mkdir -p gpurun_out
python scripts/leak_probe.py > gpurun_out/leak_probe2.txt 2>&1
python scripts/small_batch.py cfg1 > gpurun_out/small_cfg1.txt 2>&1
python scripts/small_batch.py cfg2 50000,100000,200000,333334,500000,1000000 > gpurun_out/small_cfg2.txt 2>&1
cat gpurun_out/leak_probe2.txt gpurun_out/small_cfg1.txt gpurun_out/small_cfg2.txt
