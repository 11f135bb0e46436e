import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_18052_b200 as lbg
n = int(sys.argv[1])
rng = np.random.default_rng(1)
a = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * 0.3 / n
from scipy.linalg import expm
p = lbg.expm(a, 1.0)
print(n, np.abs(p - expm(a)).max(), flush=True)
