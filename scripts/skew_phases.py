import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1107_3622_b200 as K
from paper_1107_3622_b200 import _lib
from paper_1107_3622_b200.sort_core import _sort_device
from tests.test_gpu_parity import _skewed
n = 10_000_000
for kind in ("uniform", "lognormal", "clusters"):
    rng = np.random.default_rng(1)
    a = rng.random(n) if kind == "uniform" else _skewed(kind, n, rng)
    p = torch.as_tensor(a).cuda(); k = torch.empty_like(p)
    for r in range(3):
        k.copy_(p); torch.cuda.synchronize()
        st = _sort_device(k, _lib.KS_FLAG_PROFILE)
    print(kind, {nm: round(st.phase_ms[i] * 1000, 1) for i, nm in enumerate(_lib.PHASES) if st.phase_launches[i]}, "levels", st.levels)
