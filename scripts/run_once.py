"""One warm-up sort + one measured sort of the C0 workload (for whole-sort ncu captures: use -s <launches of the first>)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1107_3622_b200 as K  # noqa: E402

n = int(os.environ.get("EXP_N", "10000000"))
pristine = K.generate_device(n, 20260816, os.environ.get("EXP_KIND", "uniform01"))
keys = torch.empty_like(pristine)
for _ in range(2):
    keys.copy_(pristine)
    torch.cuda.synchronize()
    K.k_sort(keys)
torch.cuda.synchronize()
print("sorted", bool(K.is_sorted(keys)), K.last_stats)
