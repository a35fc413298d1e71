import sys; sys.path.insert(0,".")
import numpy as np, paper_1505_01466_b200 as pb
N, k, L, fpw, sp = [int(x) for x in sys.argv[1:6]]
spec = pb.CodeSpec.from_design_ebn0(N, k, pb.CRC32, 3.0)
sch = pb.build_schedule(spec)
fb = pb.generate_frames(spec, 3.0, seed=11, start=0, count=200)
ref = pb.ListDecoder(sch, L, options={"specialize": -1}).decode_batch(fb.llrs)
d = pb.ListDecoder(sch, L, options={"frames_per_warp": fpw, "specialize": sp})
r = d.decode_batch(fb.llrs); print(sys.argv[1:], "ok", np.array_equal(r.info_bits, ref.info_bits), np.array_equal(r.chosen_pm, ref.chosen_pm))
