# e2e pipeline schedules on cfg2 (MREP_E2E_* knobs of mrep_host.cu)
mkdir -p gpurun_out
out=gpurun_out/e2e_sweep.txt
: > $out
for v in "MREP_X=0" "MREP_E2E_CONC=1" "MREP_E2E_CONC=2" "MREP_E2E_CONC=3" \
         "MREP_E2E_FIRST=65536,MREP_E2E_GEOM=2" "MREP_E2E_FIRST=65536,MREP_E2E_GEOM=2,MREP_E2E_CONC=2" \
         "MREP_E2E_FIRST=100000,MREP_E2E_GEOM=1.5" "MREP_E2E_FIRST=100000,MREP_E2E_GEOM=1.5,MREP_E2E_CONC=2" \
         "MREP_E2E_FIRST=131072,MREP_E2E_GEOM=1.3,MREP_E2E_CONC=3" "MREP_E2E_FIRST=50000,MREP_E2E_GEOM=1.6,MREP_E2E_CONC=2" \
         "MREP_E2E_FIRST=32768,MREP_E2E_GEOM=2.2,MREP_E2E_CONC=1" "MREP_E2E_CHUNK=131072" "MREP_E2E_CHUNK=131072,MREP_E2E_CONC=2" \
         "MREP_E2E_CHUNK=100000,MREP_E2E_CONC=3" "MREP_E2E_PRIO=0"; do
  envs=$(echo $v | tr ',' ' ')
  echo "$v: $(env $envs python scripts/e2e_time.py ${CFG:-cfg2} 30 2>&1 | tail -1)" >> $out
done
for v in "MREP_X=0" "MREP_E2E_FIRST=65536,MREP_E2E_GEOM=2,MREP_E2E_CONC=2" "MREP_E2E_FIRST=100000,MREP_E2E_GEOM=1.5,MREP_E2E_CONC=2"; do
  envs=$(echo $v | tr ',' ' ')
  echo "== $v" >> gpurun_out/e2e_trace2.txt
  env $envs python scripts/e2e_trace.py ${CFG:-cfg2} 3 2>&1 | grep -v "host launch" | tail -12 >> gpurun_out/e2e_trace2.txt
done
cat $out
