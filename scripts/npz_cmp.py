"""Bitwise comparison of two npz dumps."""
import sys

import numpy as np

a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
for k in a.files:
    x, y = a[k], b[k]
    same = np.array_equal(x.view(np.uint8), y.view(np.uint8))
    print(k, "identical" if same else f"DIFF {np.count_nonzero(x != y)} / {x.size}")
