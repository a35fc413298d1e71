"""Parity at volume against committed oracle digests.

``tests/golden/parity_digests.json`` holds, per BASELINE operating point, a
sha256 digest of the oracle's outputs (payload bits, CRC flag, chosen metric,
paths used) for every 4096-frame chunk of the seeded reference frame stream
-- 2^16 .. 2^20 frames per point, made by ``tools/parity_full.py oracle``
from the C restatement of listdec.py (pinned to the reference by
tests/test_oracle.py).  Here the GPU decodes the first chunks of every point
and must reproduce the digests bit for bit; ``tools/parity_full.py gpu``
runs every chunk (profiles/*_parity_full.json)."""

import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "tools"))

import parity_full  # noqa: E402

with open(parity_full.DIGESTS) as fh:
    DIGESTS = json.load(fh)


def test_digest_file_covers_the_baseline_points():
    names = set(DIGESTS)
    for pt in parity_full._points():
        assert pt in names, pt
    for name, rec in DIGESTS.items():
        assert len(rec["digests"]) * rec["chunk"] == rec["frames"]
    assert DIGESTS["c4_int8_L32_4.0"]["frames"] == 1 << 20
    assert all(DIGESTS[f"c3_L{L}_{e}"]["frames"] == 1 << 18 for L in (2, 8, 32) for e in (3.5, 4.0, 4.5))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(DIGESTS))
def test_gpu_matches_oracle_digests(name):
    chunks = 4 if name.startswith("c4") else 2
    ok = parity_full.run_gpu([name], chunks, None, min(8, os.cpu_count() or 1))
    assert ok, f"{name}: GPU output differs from the oracle digests"
