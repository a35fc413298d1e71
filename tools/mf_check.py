import sys, json; sys.path.insert(0, ".")
import numpy as np, bench, paper_1505_01466_b200 as pb
def same(a, b): return all(np.array_equal(getattr(a,f), getattr(b,f)) for f in ("info_bits","crc_ok","chosen_pm","paths_used"))
for cfg, fpw in (("c3_L8", 4), ("c3_L2", 16), ("c1_L4", 8), ("c2_L8", 4), ("c3_L8", 2)):
    spec, sch, L, ebn0, mode, label = bench.make_code(cfg)
    fb = pb.generate_frames(spec, ebn0 - 0.5, seed=11, start=0, count=1001)
    ref = pb.ListDecoder(sch, L, mode=mode, options={"specialize": -1}).decode_batch(fb.llrs)
    d = pb.ListDecoder(sch, L, mode=mode, options={"frames_per_warp": fpw, "specialize": 1})
    got = d.decode_batch(fb.llrs)
    bad = np.flatnonzero(~(np.all(got.info_bits == ref.info_bits, axis=1) & (got.chosen_pm == ref.chosen_pm) & (got.crc_ok == ref.crc_ok)))
    print(cfg, fpw, same(got, ref), bad[:10], json.loads(d.plan)["lane_kernel"])
    one = d.decode_batch(fb.llrs[3:4]); print("  single", np.array_equal(one.info_bits[0], ref.info_bits[3]))
