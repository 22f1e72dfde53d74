# e2e pipeline shapes (cfg2): default (5 equal chunks on priority streams) vs
# uniform chunk sizes (MREP_E2E_CHUNK) and the short-edge schedule (MREP_E2E_EDGE)
for rep in 1 2; do
  python scripts/diag_e2e.py cfg2 2>&1 | grep seg=False | sed "s/^/default /"
  for c in 131072 166667 250000; do
    MREP_E2E_CHUNK=$c python scripts/diag_e2e.py cfg2 2>&1 | grep seg=False
  done
  for e in 131072 196608; do
    MREP_E2E_EDGE=$e python scripts/diag_e2e.py cfg2 2>&1 | grep seg=False | sed "s/^/edge=$e /"
  done
done
