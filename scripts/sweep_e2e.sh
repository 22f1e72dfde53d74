python scripts/diag_sizes.py 65536 125000 250000 375000 500000 1000000
for s in 1 2 3; do
  for e in 65536 131072 196608; do MREP_E2E_SLOTS=$s MREP_E2E_EDGE=$e python scripts/diag_e2e.py cfg2 2>&1 | grep seg=False | sed "s/^/slots=$s edge=$e /"; done
  for c in 131072 250000 333334; do MREP_E2E_SLOTS=$s MREP_E2E_CHUNK=$c python scripts/diag_e2e.py cfg2 2>&1 | grep seg=False | sed "s/^/slots=$s /"; done
done
