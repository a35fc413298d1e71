"""Device-resident decode rate of an ad-hoc code: python tools/quick_rate.py N k L mode [opt=val ...]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1505_01466_b200 as pb
N, k, L, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
opts = {a.split("=")[0]: int(a.split("=")[1]) for a in sys.argv[5:]}
spec = pb.CodeSpec.from_design_ebn0(N, k, pb.CRC32, 3.5)
sch = pb.build_schedule(spec)
B = 32768 if N <= 2048 else 8192
fb = pb.generate_frames(spec, 3.5, seed=1, start=0, count=4096)
llr = np.tile(fb.llrs, (B // 4096, 1))
feed = llr if mode == "f32" else pb.quantize_int8(llr)
x = torch.from_numpy(feed).cuda()
dec = pb.ListDecoder(sch, L, mode=mode, options=opts)
info = torch.empty((B, spec.k), dtype=torch.uint8, device="cuda")
for _ in range(3):
    dec.decode_device(x, info)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    dec.decode_device(x, info)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(sys.argv[1:], round(B * spec.k / ms / 1e6, 3), "Gbit/s")
