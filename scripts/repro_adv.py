import sys, time, faulthandler; faulthandler.enable()
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1107_3622_b200 as K
n = int(sys.argv[1]); kind = sys.argv[2]
p = K.generate_device(n, 20260816)
if kind == "presorted": p = torch.sort(p).values
elif kind == "reversed": p = torch.sort(p, descending=True).values
elif kind == "organ":
    s = torch.sort(p).values; p = torch.cat([s[0::2], s[1::2].flip(0)])
want = torch.sort(p).values
k = torch.empty_like(p)
for call in range(4):
    k.copy_(p); torch.cuda.synchronize()
    t0 = time.time(); K.k_sort(k); torch.cuda.synchronize()
    print(n, kind, call, "%.2f ms" % ((time.time() - t0) * 1e3), bool(torch.equal(k, want)), K.last_stats, flush=True)
