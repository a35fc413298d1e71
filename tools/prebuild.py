"""Compile the specialised lane kernels of the bench / BASELINE configurations
into the in-tree cubin cache (NVRTC, no GPU needed): python tools/prebuild.py [cfg ...] [--opt k=v]"""
import sys, time
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, ".")
import bench
import paper_1505_01466_b200 as pb

opts = {}
cfgs = []
args = sys.argv[1:]
while args:
    a = args.pop(0)
    if a == "--opt":
        k, v = args.pop(0).split("=")
        opts[k] = int(v)
    else:
        cfgs.append(a)
cfgs = cfgs or ["c3_L32", "c4_int8_L32"]


def one(cfg):
    spec, sch, L, ebn0, mode, label = bench.make_code(cfg)
    t = time.time()
    hit, secs = pb.prebuild_specialised(sch, L, mode=mode, options=opts)
    return cfg, hit, round(secs, 1), pb.specialised_source(sch, L, mode=mode, options=opts)[1]


with ThreadPoolExecutor(len(cfgs)) as ex:
    for r in ex.map(one, cfgs):
        print(*r)
