import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1107_3622_b200 as K
from tests.test_gpu_parity import _skewed
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
rng = np.random.default_rng(hash(("bit_patterns", n)) % 2**32)
a = _skewed("bit_patterns", n, rng)
t = torch.as_tensor(a).cuda()
K.k_sort(t)
r = t.cpu().numpy(); e = np.sort(a)
print(n, "mismatches", int(np.sum(r.view(np.int64) != e.view(np.int64))), K.last_stats)
