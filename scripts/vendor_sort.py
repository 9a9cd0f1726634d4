"""Context only (not the product, not a target): torch.sort (CUB radix sort) on the C0 workload."""
import torch
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_3622_b200 as K
n = 10_000_000
x = K.generate_device(n, 20260816)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for name, fn in (("torch.sort(values+indices)", lambda t: torch.sort(t)), ("ksort", lambda t: K.k_sort(t))):
    ts = []
    for i in range(8):
        y = x.clone(); flush.zero_(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(y); b.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b))
    print("%-28s %.3f ms  %.2f G keys/s" % (name, min(ts), n / min(ts) / 1e6))
