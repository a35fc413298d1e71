#!/usr/bin/env python3
"""Full-volume parity at BASELINE volumes (SURVEY.md 8(d) parity criteria).

Two legs over the same seeded input streams (the reference harness's own
per-frame Philox generator, ``channel.generate_frames`` == reference
``sim.py:73-91``):

  oracle   CPU: decode every chunk of 4096 frames with the C restatement of
           ``listdec.py`` (``oracle/``, all host threads) and record one
           digest per chunk -- sha256 of (packed info bits | crc_ok |
           chosen_pm float64 | paths_used int32) -- plus frame / bit error
           counts.  Output: ``tests/golden/parity_digests.json``.
  gpu      the B200 decoder on the same frames: per-chunk digests compared
           with the committed oracle digests; a mismatching chunk is bisected
           to frames.  Reports FER / BER with the reference's 95 % Wilson
           interval (``pkg/tests/test_acceptance.py:222-230``).
           Output: ``profiles/<tag>_parity_full.json``.

Seeds: 1000 * config index + round(10 * Eb/N0).

  python tools/parity_full.py oracle [--points c3_L32_4.0,...] [--threads 8]
  python tools/parity_full.py gpu [--max-chunks K] [--out profiles/x.json]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_1505_01466_b200 as pb  # noqa: E402

CHUNK = 4096
DIGESTS = os.path.join(REPO, "tests", "golden", "parity_digests.json")


def _points():
    """(name, cfg index, N, K incl. CRC, crc, design Eb/N0, L, Eb/N0, mode, frames)."""
    crc8 = ("crc8_d5", 8)
    crc32 = ("crc32", 32)
    pts = [("c1_L4_2.5", 1, 1024, 512, crc8, 2.0, 4, 2.5, "f32", 4096)]
    for e in (3.5, 4.0, 4.5):
        pts.append((f"c2_L8_{e}", 2, 1024, 860, crc32, 4.0, 8, e, "f32", 1 << 16))
    for L in (2, 8, 32):
        for e in (3.5, 4.0, 4.5):
            pts.append((f"c3_L{L}_{e}", 3, 2048, 1723, crc32, 4.0, L, e, "f32", 1 << 18))
    pts.append(("c4_int8_L32_4.0", 4, 2048, 1723, crc32, 4.0, 32, 4.0, "int8", 1 << 20))
    pts.append(("c5_L16_3.0", 5, 8192, 6144, crc32, 3.0, 16, 3.0, "f32", 1 << 16))
    return {p[0]: p for p in pts}


def _crc(name):
    return pb.CrcConfig(width=8, polynomial=0xD5) if name == "crc8_d5" else pb.CRC32


def _code(pt):
    _, ci, N, K, (crc_name, w), design, L, ebn0, mode, frames = pt
    spec = pb.CodeSpec.from_design_ebn0(N, K - w, _crc(crc_name), design)
    return spec, pb.build_schedule(spec), L, ebn0, mode, frames, 1000 * ci + int(round(10 * ebn0))


def digest(info_bits, crc_ok, pm, paths_used) -> str:
    h = hashlib.sha256()
    h.update(np.packbits(np.asarray(info_bits, np.uint8), axis=1).tobytes())
    h.update(np.asarray(crc_ok, np.uint8).tobytes())
    h.update(np.asarray(pm, "<f8").tobytes())
    h.update(np.asarray(paths_used, "<i4").tobytes())
    return h.hexdigest()[:32]


def errors(info_bits, payloads):
    d = np.asarray(info_bits, np.uint8) != np.asarray(payloads, np.uint8)
    return int(d.any(axis=1).sum()), int(d.sum())


def wilson(errors_, frames):
    """95 % Wilson score interval (reference pkg/tests/test_acceptance.py:222-230)."""
    if frames == 0:
        return 0.0, 1.0
    z = 1.96
    p = errors_ / frames
    denom = 1.0 + z * z / frames
    center = (p + z * z / (2 * frames)) / denom
    half = z * math.sqrt(p * (1 - p) / frames + z * z / (4 * frames ** 2)) / denom
    return center - half, center + half


def _blocks(spec, nch, workers):
    """Frame batches of whole chunks (a few chunks per generator pool)."""
    per = max(1, (1 << 26) // (spec.N * 4 * CHUNK))
    for c0 in range(0, nch, per):
        cn = min(per, nch - c0)
        yield c0, cn


def run_oracle(names, threads):
    from oracle import oracle
    out = {}
    if os.path.exists(DIGESTS):
        with open(DIGESTS) as fh:
            out = json.load(fh)
    pts = _points()
    for name in names:
        spec, sch, L, ebn0, mode, frames, seed = _code(pts[name])
        t0 = time.time()
        rec = {"N": spec.N, "k": spec.k, "L": L, "ebn0": ebn0, "mode": mode, "seed": seed,
               "frames": frames, "chunk": CHUNK, "digests": [], "frame_errors": 0, "bit_errors": 0}
        for c0, cn in _blocks(spec, frames // CHUNK, threads):
            fb = pb.generate_frames(spec, ebn0, seed=seed, start=c0 * CHUNK, count=cn * CHUNK,
                                    workers=threads)
            feed = pb.quantize_int8(fb.llrs) if mode == "int8" else fb.llrs  # the oracle's int8 mode takes quantised LLRs
            r = oracle.decode_batch(sch, L, feed, int8=(mode == "int8"), threads=threads)
            for j in range(cn):
                s = slice(j * CHUNK, (j + 1) * CHUNK)
                rec["digests"].append(digest(r.info_bits[s], r.crc_ok[s], r.chosen_pm[s],
                                             r.paths_used[s]))
                fe, be = errors(r.info_bits[s], fb.payloads[s])
                rec["frame_errors"] += fe
                rec["bit_errors"] += be
        rec["oracle_s"] = round(time.time() - t0, 1)
        out[name] = rec
        print(f"{name}: {frames} frames, FER {rec['frame_errors'] / frames:.3e}, "
              f"{rec['oracle_s']} s", flush=True)
        with open(DIGESTS, "w") as fh:
            json.dump(out, fh, indent=1)


def run_gpu(names, max_chunks, out_path, workers):
    with open(DIGESTS) as fh:
        ref = json.load(fh)
    pts = _points()
    report = {"chunk": CHUNK, "points": {}}
    all_ok = True
    for name in names:
        if name not in ref:
            continue
        r0 = ref[name]
        spec, sch, L, ebn0, mode, frames, seed = _code(pts[name])
        dec = pb.ListDecoder(sch, L, mode=mode)
        nch = len(r0["digests"]) if max_chunks is None else min(max_chunks, len(r0["digests"]))
        bad, fe_tot, be_tot, t_gen, t_dec = [], 0, 0, 0.0, 0.0
        for c0, cn in _blocks(spec, nch, workers):
            t = time.time()
            fbb = pb.generate_frames(spec, ebn0, seed=seed, start=c0 * CHUNK, count=cn * CHUNK,
                                     workers=workers)
            t_gen += time.time() - t
            t = time.time()
            rb = dec.decode_batch(fbb.llrs)
            t_dec += time.time() - t
            for j in range(cn):
                s = slice(j * CHUNK, (j + 1) * CHUNK)
                c = c0 + j
                d = digest(rb.info_bits[s], rb.crc_ok[s], rb.chosen_pm[s], rb.paths_used[s])
                fe, be = errors(rb.info_bits[s], fbb.payloads[s])
                fe_tot += fe
                be_tot += be
                if d != r0["digests"][c]:
                    bad.append(_bisect(sch, L, mode, fbb.llrs[s], rb, s, c))
        n = nch * CHUNK
        lo, hi = wilson(fe_tot, n)
        ok = not bad
        all_ok &= ok
        entry = {"frames": n, "chunks": nch, "chunks_identical": nch - len(bad),
                 "mismatching_chunks": bad, "frame_errors": fe_tot, "bit_errors": be_tot,
                 "fer": fe_tot / n, "ber": be_tot / (n * spec.k), "fer_wilson95": [lo, hi],
                 "gen_s": round(t_gen, 1), "decode_s": round(t_dec, 2)}
        if nch == len(r0["digests"]):
            entry["oracle_frame_errors"] = r0["frame_errors"]
            entry["oracle_bit_errors"] = r0["bit_errors"]
            olo, ohi = wilson(r0["frame_errors"], n)
            entry["oracle_fer_wilson95"] = [olo, ohi]
        report["points"][name] = entry
        print(f"{name}: {nch - len(bad)}/{nch} chunks identical, FER {fe_tot / n:.3e} "
              f"[{lo:.2e}, {hi:.2e}]", flush=True)
    report["all_identical"] = all_ok
    if out_path:
        with open(out_path, "w") as fh:
            json.dump(report, fh, indent=1)
    return all_ok


def _bisect(sch, L, mode, llrs, rb, s, c):
    """Frames of a mismatching chunk that differ from the oracle."""
    from oracle import oracle
    feed = pb.quantize_int8(llrs) if mode == "int8" else llrs
    o = oracle.decode_batch(sch, L, feed, int8=(mode == "int8"), threads=os.cpu_count() or 1)
    ib, ok, pm, pu = rb.info_bits[s], rb.crc_ok[s], rb.chosen_pm[s], rb.paths_used[s]
    diff = np.nonzero((o.info_bits != ib).any(axis=1) | (o.crc_ok != ok)
                      | (o.chosen_pm != pm) | (o.paths_used != pu))[0]
    return {"chunk": c, "frames": [int(c * CHUNK + i) for i in diff[:64]],
            "bits_differ": int((o.info_bits != ib).any(axis=1).sum()),
            "max_pm_diff": float(np.max(np.abs(o.chosen_pm - pm))) if len(diff) else 0.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("leg", choices=["oracle", "gpu"])
    ap.add_argument("--points", default="all")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--max-chunks", type=int, default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    names = list(_points()) if a.points == "all" else a.points.split(",")
    if a.leg == "oracle":
        run_oracle(names, a.threads)
    else:
        ok = run_gpu(names, a.max_chunks, a.out, a.threads)
        sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
