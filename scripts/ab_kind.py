import ctypes, os, sys, statistics, zlib
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1107_3622_b200 import _lib
import paper_1107_3622_b200 as K
from tests.test_gpu_parity import _skewed
n = int(sys.argv[1]); kind = sys.argv[2]
rng = np.random.default_rng(1)
p = torch.as_tensor(_skewed(kind, n, rng)).cuda(); want = torch.sort(p).values
flush = torch.empty(256*1024*1024//8, dtype=torch.float64, device="cuda")
for path in sys.argv[3:]:
    L = ctypes.CDLL(os.path.abspath(path))
    L.ks_workspace_bytes.argtypes=[ctypes.c_int64,ctypes.c_int64,ctypes.c_uint32]; L.ks_workspace_bytes.restype=ctypes.c_size_t
    L.ks_sort_f64.argtypes=[ctypes.c_void_p,ctypes.c_int64,ctypes.c_void_p,ctypes.c_size_t,ctypes.c_void_p,ctypes.c_uint32,ctypes.POINTER(_lib.KsStatus)]
    wsb=L.ks_workspace_bytes(n,1,0); ws=torch.empty(wsb,dtype=torch.uint8,device="cuda"); st=_lib.KsStatus(); k=torch.empty_like(p); ts=[]
    for r in range(8):
        k.copy_(p); flush.zero_(); torch.cuda.synchronize()
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); rc=L.ks_sort_f64(k.data_ptr(),n,ws.data_ptr(),wsb,torch.cuda.current_stream().cuda_stream,0,ctypes.byref(st)); e1.record(); torch.cuda.synchronize()
        if r>=3: ts.append(e0.elapsed_time(e1))
    print(kind, n, os.path.basename(path), round(statistics.median(ts),3), "levels", st.levels, "syncs", st.host_syncs, "ok", bool(torch.equal(k,want)), flush=True)
