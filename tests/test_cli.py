"""CLI (reference cli.py): host-side subcommands and exit codes on CPU; the
GPU subcommands (decode / simulate / bench) under -m gpu."""

import numpy as np
import pytest

import paper_1505_01466_b200 as pb
from paper_1505_01466_b200 import cli


def test_usage_and_errors(tmp_path, capsys):
    assert cli.main([]) == 1
    assert cli.main(["nosuch"]) == 1
    assert cli.main(["emit", "--spec", str(tmp_path / "missing.txt")]) == 2
    assert "error:" in capsys.readouterr().err
    assert cli.parse_snr("1:2:0.5") == [1.0, 1.5, 2.0]
    with pytest.raises(ValueError):
        cli.parse_snr("1:2")


def test_construct_encode_emit_round_trip(tmp_path):
    spec_p = tmp_path / "spec.txt"
    assert cli.main(["construct", "--n", "64", "--k", "28", "--crc", "8", "--out", str(spec_p)]) == 0
    spec = pb.CodeSpec.load(str(spec_p))
    assert spec.N == 64 and spec.k == 28 and spec.crc.width == 8
    rng = np.random.default_rng(1)
    pays = rng.integers(0, 2, (5, 28), dtype=np.uint8)
    cli.write_bit_lines(tmp_path / "pay.txt", pays)
    assert cli.main(["encode", "--spec", str(spec_p), "--in", str(tmp_path / "pay.txt"),
                     "--out", str(tmp_path / "cw.txt")]) == 0
    cws = cli.read_bit_lines(tmp_path / "cw.txt")
    for p, c in zip(pays, cws):
        assert np.array_equal(c, pb.attach_and_encode(p, spec).codeword)
    assert cli.main(["emit", "--spec", str(spec_p), "--out", str(tmp_path / "e.txt")]) == 0
    assert (tmp_path / "e.txt").read_text() == pb.emit_source(pb.build_schedule(spec))


def test_bench_rejects_the_per_bit_variant(tmp_path, capsys):
    spec_p = tmp_path / "spec.txt"
    cli.main(["construct", "--n", "64", "--k", "28", "--crc", "8", "--out", str(spec_p)])
    assert cli.main(["bench", "--spec", str(spec_p), "--variants", "scl", "--list", "2"]) == 2


@pytest.mark.gpu
def test_gpu_decode_simulate_bench(tmp_path, capsys):
    spec_p = tmp_path / "spec.txt"
    cli.main(["construct", "--n", "256", "--k", "120", "--crc", "32", "--out", str(spec_p)])
    spec = pb.CodeSpec.load(str(spec_p))
    fb = pb.generate_frames(spec, 3.0, 4, 0, 20, workers=1)
    with open(tmp_path / "llr.txt", "w") as fh:
        for x in fb.llrs:
            fh.write(" ".join(repr(float(v)) for v in x) + "\n")
    from oracle import oracle
    sch = pb.build_schedule(spec)
    parsed = pb.clamp_llr(np.stack(cli.read_llr_lines(tmp_path / "llr.txt")))
    for extra in ([], ["--adaptive"]):
        assert cli.main(["decode", "--spec", str(spec_p), "--list", "8", "--in", str(tmp_path / "llr.txt"),
                         "--out", str(tmp_path / "dec.txt"), *extra]) == 0
        got = np.stack(cli.read_bit_lines(tmp_path / "dec.txt"))
        assert got.shape == (20, 120)
        # the CPU oracle (restatement of the reference, pinned to its fixtures)
        exp = (oracle.adaptive_batch(sch, 8, parsed) if extra else oracle.decode_batch(sch, 8, parsed))
        assert np.array_equal(got, exp.info_bits), extra
    assert cli.main(["simulate", "--spec", str(spec_p), "--list", "4", "--snr", "1:2:1", "--min-errors", "5",
                     "--max-frames", "2000", "--out", str(tmp_path / "s.csv")]) == 0
    lines = (tmp_path / "s.csv").read_text().splitlines()
    assert len(lines) == 3 and lines[0].startswith("snr_db,frames")
    assert cli.main(["simulate", "--spec", str(spec_p), "--snr", "2", "--frames", "device", "--min-errors", "0",
                     "--max-frames", "5000", "--adaptive", "--list", "4"]) == 0
    capsys.readouterr()
    assert cli.main(["bench", "--spec", str(spec_p), "--list", "2,8", "--frames", "3"]) == 0
    out = capsys.readouterr().out
    assert "spc4+" in out and "unrolled" in out
