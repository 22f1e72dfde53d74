# e2e pipeline shapes (cfg2): default edge schedule, uniform chunks, priority on/off
for pr in 1 0; do
  MREP_E2E_PRIO=$pr python scripts/diag_e2e.py cfg2 2>&1 | grep seg=False | sed "s/^/prio=$pr default /"
  for c in 65536 100000 131072 200000 250000; do
    MREP_E2E_PRIO=$pr MREP_E2E_SLOTS=4 MREP_E2E_CHUNK=$c python scripts/diag_e2e.py cfg2 2>&1 | grep seg=False | sed "s/^/prio=$pr /"
  done
  for e in 65536 98304 196608; do
    MREP_E2E_PRIO=$pr MREP_E2E_EDGE=$e python scripts/diag_e2e.py cfg2 2>&1 | grep seg=False | sed "s/^/prio=$pr edge=$e /"
  done
done
MREP_E2E_TRACE=1 MREP_E2E_SLOTS=4 MREP_E2E_CHUNK=131072 python scripts/diag_e2e.py cfg2 2>&1 | tail -9
