# e2e pipeline shapes (cfg2): default edge schedule vs uniform chunks (priority streams)
for rep in 1 2; do
  python scripts/diag_e2e.py cfg2 2>&1 | grep seg=False | sed "s/^/default /"
  for c in 100000 131072 166667 200000 250000; do
    MREP_E2E_SLOTS=4 MREP_E2E_CHUNK=$c python scripts/diag_e2e.py cfg2 2>&1 | grep seg=False
  done
  for e in 98304 131072 196608; do
    MREP_E2E_EDGE=$e python scripts/diag_e2e.py cfg2 2>&1 | grep seg=False | sed "s/^/edge=$e /"
  done
done
