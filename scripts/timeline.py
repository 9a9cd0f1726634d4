"""Per-item timeline of the leaf phase (exp/lib_tl.so, built with -DKS_TIMELINE):

    bash scripts/exp_build.sh tl "-DKS_TIMELINE"
    python scripts/timeline.py [n] [kind] [out.json]

Records {sm, kernel, kind, len, t0, t1} (globaltimer ns) of every leaf item and
every persistent CTA of k_leaf / k_segsort; prints per-kernel spans, CTA busy
fractions, the item-size histogram and the critical tail of k_leaf.
kernel: 2 = k_leaf, 10 + C = k_segsort<C>; kind: 0 fetch/wait, 1 local
partition (k_leaf) or sort, 2 sort (k_leaf), 9 whole CTA.
"""
import ctypes
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("KSORT_LIB", os.path.join(ROOT, "exp", "lib_tl.so"))
from paper_1107_3622_b200 import _lib  # noqa: E402
import torch  # noqa: E402
import paper_1107_3622_b200 as K  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
kind = sys.argv[2] if len(sys.argv) > 2 else "uniform01"
out = sys.argv[3] if len(sys.argv) > 3 else None
L = _lib.load()
L.ks_timeline_read.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
L.ks_timeline_read.restype = ctypes.c_int
cap = 1 << 17
buf = (ctypes.c_ulonglong * (4 * cap))()
p = K.generate_device(n, 20260816, kind)
k = torch.empty_like(p)
flush = torch.empty(int(os.environ.get("TL_FLUSH_MB", "256")) * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
L.ks_timeline_mark.argtypes = [ctypes.c_void_p, ctypes.c_int]
sp = torch.cuda.current_stream().cuda_stream
for rep in range(4):
    k.copy_(p)
    flush.zero_()
    torch.cuda.synchronize()
    L.ks_timeline_read(None, 0, 1)
    flush.zero_()                 # (the GPU is busy while the call is issued, as in bench.py)
    L.ks_timeline_mark(sp, 30)    # mark: the flush has ended
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record()
    K.k_sort(k)
    eb.record()
    L.ks_timeline_mark(sp, 31)    # mark: enqueued after the call returned
    torch.cuda.synchronize()
    ev_ms = ea.elapsed_time(eb)
m = L.ks_timeline_read(ctypes.addressof(buf), cap, 0)
assert torch.equal(k, torch.sort(p).values)
recs = []
for i in range(m):
    w = buf[4 * i]
    recs.append({"sm": w & 0xff, "kernel": (w >> 8) & 0xff, "kind": ((w >> 16) & 0xff) - 1, "len": buf[4 * i + 1],
                 "t0": buf[4 * i + 2], "t1": buf[4 * i + 3]})
T0 = min(r["t0"] for r in recs)
for r in recs:
    r["t0"] -= T0
    r["t1"] -= T0
names = {30: "mark0", 31: "mark1", 2: "k_leaf", 10: "segsort<0>", 11: "segsort<1>", 13: "segsort<3>", 14: "segsort<4>", 20: "init_pass", 22: "front_lut",
         21: "pivot_rank", 23: "count2", 24: "scan", 25: "plan", 26: "scatter2", 27: "leaf_reset", 40: "small:rank", 41: "small:count", 42: "small:scatter",
         43: "small:sort", 44: "small:barrier"}
print(f"n={n} kind={kind} records={m} event span {ev_ms*1e3:.1f} us")
mk = {r["kernel"]: r for r in recs if r["kernel"] in (30, 31)}
if 30 in mk and 31 in mk:
    first = min(r["t0"] for r in recs if r["kernel"] not in (30, 31))
    last = max(r["t1"] for r in recs if r["kernel"] not in (30, 31))
    print(f"  mark(before) end {mk[30]['t1']/1e3:.1f} us -> first kernel {first/1e3:.1f} us; last kernel end "
          f"{last/1e3:.1f} us -> mark(after) start {mk[31]['t0']/1e3:.1f} us")
for kern in sorted({r["kernel"] for r in recs}):
    cta = [r for r in recs if r["kernel"] == kern and r["kind"] == 8]
    items = [r for r in recs if r["kernel"] == kern and r["kind"] in (0, 1)]
    if kern == 2:
        items = [r for r in recs if r["kernel"] == kern and r["kind"] in (0, 1) and True]
    if not cta:
        continue
    if kern >= 20:
        s0, s1 = min(r["t0"] for r in cta), max(r["t1"] for r in cta)
        ends = sorted(r["t1"] for r in cta)
        print(f"{names.get(kern, kern):12s} span {s0/1e3:7.1f}..{s1/1e3:7.1f} us ({(s1-s0)/1e3:6.1f})  CTAs {len(cta):4d}  "
              f"CTA end p50 {ends[len(ends)//2]/1e3:.1f}")
        continue
    s0, s1 = min(r["t0"] for r in cta), max(r["t1"] for r in cta)
    busy = sum(r["t1"] - r["t0"] for r in recs if r["kernel"] == kern and r["kind"] in (0, 1) and kern != 2) if kern != 2 \
        else sum(r["t1"] - r["t0"] for r in recs if r["kernel"] == 2 and r["kind"] in (0, 1))
    ctat = sum(r["t1"] - r["t0"] for r in cta)
    ends = sorted(r["t1"] for r in cta)
    print(f"{names.get(kern, kern):12s} span {s0/1e3:7.1f}..{s1/1e3:7.1f} us ({(s1-s0)/1e3:6.1f})  CTAs {len(cta):4d}  "
          f"CTA-time {ctat/1e3:8.1f} us  items-busy {busy/ctat*100:5.1f}%  CTA end p10/p50/p90 "
          f"{ends[len(ends)//10]/1e3:.1f}/{ends[len(ends)//2]/1e3:.1f}/{ends[9*len(ends)//10]/1e3:.1f}")
# k_leaf detail
lf = [r for r in recs if r["kernel"] == 2]
if lf:
    fetch = [r for r in lf if r["kind"] == -1]
    loc = [r for r in lf if r["kind"] == 0]
    srt = [r for r in lf if r["kind"] == 1]
    tot = sum(r["t1"] - r["t0"] for r in lf if r["kind"] == 8)
    f = lambda rs: sum(r["t1"] - r["t0"] for r in rs)
    print(f"k_leaf CTA-time split: fetch/wait {f(fetch)/tot*100:.1f}%  local {f(loc)/tot*100:.1f}% ({len(loc)} items, "
          f"{sum(r['len'] for r in loc)} keys)  sort {f(srt)/tot*100:.1f}% ({len(srt)} items, {sum(r['len'] for r in srt)} keys)")
    if loc:
        ns_per_key = f(loc) / sum(r["len"] for r in loc)
        print(f"  local: {ns_per_key:.2f} ns/key/CTA; largest: " +
              ", ".join(f"{r['len']}@{r['t0']/1e3:.0f}-{r['t1']/1e3:.0f}us" for r in sorted(loc, key=lambda r: -r["len"])[:6]))
    if srt:
        ns_per_key = f(srt) / sum(r["len"] for r in srt)
        print(f"  sort: {ns_per_key:.2f} ns/key/CTA, mean item {sum(r['len'] for r in srt)/len(srt):.0f} keys")
    # utilisation over time (fraction of 148 CTAs inside an item) in 5 us bins
    end = max(r["t1"] for r in lf if r["kind"] == 8)
    start = min(r["t0"] for r in lf if r["kind"] == 8)
    bins = defaultdict(float)
    for r in loc + srt:
        a, b = r["t0"], r["t1"]
        t = a
        while t < b:
            bi = int((t - start) // 5000)
            e = min(b, start + (bi + 1) * 5000)
            bins[bi] += e - t
            t = e
    print("  busy CTAs per 5 us bin: " + " ".join(f"{bins[i]/5000:.0f}" for i in range(int((end - start) // 5000) + 1)))
for kern in (13, 14, 11, 10):
    it = [r for r in recs if r["kernel"] == kern and r["kind"] == 1]
    if it:
        tk = sum(r["len"] for r in it)
        print(f"{names[kern]}: {len(it)} items {tk} keys, {sum(r['t1']-r['t0'] for r in it)/tk:.2f} ns/key/CTA "
              f"mean {tk/len(it):.0f} keys")
ph = [r for r in recs if r["kernel"] in (50, 51, 52)]
if ph:
    import statistics as _st
    tiles = [r for r in ph if r["kernel"] == 50]
    a = [r["len"] / 1e3 for r in ph if r["kernel"] == 51]
    b = [r["len"] / 1e3 for r in ph if r["kernel"] == 52]
    tot = [(r["t1"] - r["t0"]) / 1e3 for r in tiles]
    print(f"scatter2 tiles (CTAs 0-3): {len(tiles)}; per tile us: total {_st.mean(tot):.2f}, A table+scan "
          f"{_st.mean(a):.2f}, B staging {_st.mean(b):.2f}, C issue {_st.mean(tot) - _st.mean(a) - _st.mean(b):.2f}")
if out:
    json.dump(recs, open(out, "w"))
