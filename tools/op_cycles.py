"""Dev helper: per-op cycle profile of one frame (CTA 0, clock64)."""
import ctypes, os, sys, collections
import numpy as np
sys.path.insert(0, '.')
# needs the instrumented build: _native.build(profile=True)
os.environ.setdefault('PB_LIB_PATH', 'paper_1505_01466_b200/_lib/libpolar_b200_prof.so')
import paper_1505_01466_b200 as pb
from paper_1505_01466_b200 import _native
import bench
cfg = sys.argv[1] if len(sys.argv) > 1 else 'c3_L32'
spec, sch, L, ebn0, mode, label = bench.make_code(cfg)
dec = pb.ListDecoder(sch, L, mode=mode)
lib = _native.lib()
lib.pb_device_op_count.restype = ctypes.c_int
lib.pb_device_op_count.argtypes = [ctypes.c_void_p]
lib.pb_profile_ops.restype = ctypes.c_int
lib.pb_profile_ops.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
n = lib.pb_device_op_count(dec._h)
fb = pb.generate_frames(spec, ebn0, seed=1, start=0, count=int(os.environ.get('OPC_FRAMES', 4096)))
llr = np.ascontiguousarray(fb.llrs)
cyc4 = np.zeros((n, 12), np.int64); kinds = np.zeros(n, np.int8); stages = np.zeros(n, np.int8)
rc = lib.pb_profile_ops(dec._h, llr.ctypes.data, 0, len(llr), cyc4.ctypes.data, kinds.ctypes.data, stages.ctypes.data)
_native.check(rc, 'pb_profile_ops')
if os.environ.get('OPC_STRIDE') == '4':  # older builds: 4 longs per op
    cyc4 = np.concatenate([cyc4.ravel()[:4 * n].reshape(n, 4), np.zeros((n, 8), np.int64)], 1)
cyc = cyc4[:, 0]
names = {0: 'F', 1: 'G', 2: 'R0', 3: 'REP', 4: 'R1', 5: 'SPC', 6: 'NOP', 7: 'FM', 8: 'GM'}
tot = cyc.sum()
print(f'{cfg}: {n} device ops, {tot} cycles for one frame (CTA 0, warps sharing the SM)')
agg = collections.defaultdict(lambda: [0, 0])
for k, s, c in zip(kinds, stages, cyc):
    agg[(names[int(k)], int(s))][0] += 1; agg[(names[int(k)], int(s))][1] += int(c)
byk = collections.defaultdict(int)
for (k, s), (cnt, c) in agg.items(): byk[k] += c
print(' '.join(f'{k}={v/tot*100:.1f}%' for k, v in sorted(byk.items(), key=lambda t: -t[1])))
for (k, s), (cnt, c) in sorted(agg.items(), key=lambda t: -t[1][1])[:25]:
    print(f'{k:4s} stage {s:2d}: {cnt:4d} ops  {c:9d} cycles  {c/cnt:8.0f}/op  {c/tot*100:5.1f}%')


# marks: 0 A end, 1 B end, 2 scan loop end, 4 B keys+sort, 5 B merge, 6 B counting, 7 C copies
t0 = cyc4[:, 1]
def rel(col):
    v = cyc4[:, 2 + col]
    return np.where(v > 0, v - t0, 0)
marks = {m: rel(m) for m in range(10)}
print('leaf timeline (mean cycles since op start): scanloop A_end keys merge count B_end C_copies end')
groups = [(kk, None) for kk in (2, 3, 4, 5)] + sorted({(int(k), int(st)) for k, st in zip(kinds, stages) if 2 <= k <= 5})
for kk, sg in groups:
    sel = (kinds == kk) & ((stages == sg) if sg is not None else True)
    if not sel.any():
        continue
    def mm(m):
        v = marks[m][sel]
        v = v[v > 0]
        return f"{v.mean():7.0f}" if v.size else "      -"
    print(f'  {names[kk]:4s}{"" if sg is None else sg:>3} n={int(sel.sum()):3d} ' + ' '.join(mm(m) for m in (2, 0, 4, 5, 6, 1, 7)) + f' {cyc4[sel,0].mean():7.0f}')

# lane kernel: cycles by active-path count (pin) bucket
try:
    import json as _json
    plan = _json.loads(dec.plan)
    if plan.get("lane_kernel"):
        n = spec.n
        cand = lambda op: (1 if op.kind is pb.NodeKind.RATE0 else 2 if (op.kind is pb.NodeKind.REP or (op.kind is pb.NodeKind.RATE1 and op.size == 1)) else 4 if op.kind is pb.NodeKind.RATE1 else (2 if L == 2 else 8))
        P, pins = 1, []
        for op in sch.ops:
            k = op.kind
            if k is pb.NodeKind.COMBINE:
                continue
            if k in (pb.NodeKind.F, pb.NodeKind.G):
                if op.stage >= n - 1 and mode == "f32" or op.stage >= n and mode != "f32":
                    continue
                pins.append(P)
                continue
            pins.append(P)
            if k is not pb.NodeKind.RATE0:
                P = min(L, P * cand(op))
        pins = np.array(pins[:len(cyc)])
        print("cycles by active paths before the op:")
        for lo, hi in ((1, 1), (2, 4), (5, 16), (17, 31), (32, 32)):
            sel = (pins >= lo) & (pins <= hi)
            print(f"  pin {lo:2d}..{hi:2d}: {sel.sum():4d} ops {cyc[:len(pins)][sel].sum():9d} cycles {100 * cyc[:len(pins)][sel].sum() / tot:5.1f}%")
except Exception as e:  # noqa: BLE001
    print("pin buckets unavailable:", e)
