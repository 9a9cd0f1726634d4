"""Sort time vs the workspace's placement relative to the keys (same library,
same input): the workspace pointer is offset by `delta` bytes inside one
allocation.  Shows whether the tmp buffer's address bits relative to the keys
matter (L2 slice / DRAM channel hashing)."""
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1107_3622_b200 import _lib  # noqa: E402
import paper_1107_3622_b200 as K  # noqa: E402

L = _lib.load()
n = int(os.environ.get("EXP_N", "10000000"))
kind = os.environ.get("EXP_KIND", "uniform01")
reps = int(os.environ.get("EXP_REPS", "15"))
pristine = K.generate_device(n, 20260816, kind)
keys = torch.empty_like(pristine)
wsb = L.ks_workspace_bytes(n, 1, 0)
big = torch.empty(wsb + (8 << 20), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
stream = torch.cuda.current_stream()
st = _lib.KsStatus()
deltas = [int(x) for x in os.environ.get("EXP_DELTAS", "0,256,4096,65536,262144,524288,1048576,1572864,2097152,3145728").split(",")]
base = big.data_ptr()
print(json.dumps({"keys_mod_2M": keys.data_ptr() % (2 << 20), "ws_mod_2M": base % (2 << 20)}))
res = {d: [] for d in deltas}
for r in range(reps + 2):
    for d in deltas:
        keys.copy_(pristine)
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rc = L.ks_sort_f64(keys.data_ptr(), n, base + d, wsb, stream.cuda_stream, 0, ctypes.byref(st))
        b.record(stream)
        torch.cuda.synchronize()
        assert rc == 0
        if r >= 2:
            res[d].append(a.elapsed_time(b))
for d in deltas:
    print(json.dumps({"delta": d, "ms_median": round(statistics.median(res[d]), 4)}))
