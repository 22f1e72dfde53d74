# ncu --set full + source of the cfg3 traversal kernel (global group walk; VARIANT=staged for the staged one)
mkdir -p gpurun_out
v=${VARIANT:-group}
k=wave_traverse_staged; env="MREP_X=0"
[ $v = group ] && { k=wave_traverse_group; env="MREP_NO_STAGE=1"; }
env $env ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
    -o gpurun_out/cfg3_$v -f python scripts/one_batch.py > gpurun_out/ncu_cfg3_$v.log 2>&1
