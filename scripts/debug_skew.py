import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1107_3622_b200 as K
from tests.test_gpu_parity import _skewed
for n in (3_000_000, 1_000_000, 600_000):
    rng = np.random.default_rng(hash(("bit_patterns", n)) % 2**32)
    a = _skewed("bit_patterns", n, rng)
    t = torch.as_tensor(a).cuda()
    K.k_sort(t)
    r = t.cpu().numpy(); e = np.sort(a)
    bad = np.nonzero(r.view(np.int64) != e.view(np.int64))[0]
    print(n, "mismatches", bad.size, "sorted?", bool(np.all(r[1:] >= r[:-1])), "multiset equal?", bool(np.array_equal(np.sort(r), e)), K.last_stats)
    if bad.size:
        print(" first/last bad", bad[:5], bad[-5:])
        i = bad[0]
        print(" got", r[i-2:i+5]); print(" exp", e[i-2:i+5])
