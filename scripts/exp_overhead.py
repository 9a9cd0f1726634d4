"""Host-side overhead inside the timed region: K.k_sort vs a bare C-ABI call with prepared arguments."""
import ctypes, os, statistics, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1107_3622_b200 as K
from paper_1107_3622_b200 import _lib
L = _lib.load()
n = 10_000_000
p = K.generate_device(n, 20260816)
k = torch.empty_like(p)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
wsb = L.ks_workspace_bytes(n, 1, 0)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
st = _lib.KsStatus()
sp = torch.cuda.current_stream().cuda_stream
def bare():
    L.ks_sort_f64(k.data_ptr(), n, ws.data_ptr(), wsb, sp, 0, ctypes.byref(st))
def api():
    K.k_sort(k)
for name, fn in (("api", api), ("bare", bare), ("api", api), ("bare", bare)):
    ts = []; hs = []
    for r in range(13):
        k.copy_(p); flush.zero_(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); t0 = time.perf_counter(); fn(); t1 = time.perf_counter(); b.record(); torch.cuda.synchronize()
        if r >= 3: ts.append(a.elapsed_time(b)); hs.append((t1 - t0) * 1e3)
    print(name, "device ms %.4f  host ms %.4f" % (statistics.median(ts), statistics.median(hs)))
