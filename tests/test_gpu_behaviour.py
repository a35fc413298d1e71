"""The reference's behavioural properties of a list decoder, re-run with the
GPU decoder substituted (the properties the reference
checks in pkg/tests/test_listdec.py:175-231 and test_acceptance.py:158-219,
restated here with independent scalar oracles written for this suite):

* exact maximum likelihood when the list holds every codeword ((8,4), L=16);
* every surviving path carries a consistent (codeword, metric) pair and a
  non-positive metric;
* a CRC-passing path beats any better-metric failing path;
* brute-force optimality of the chosen path whenever L >= 2^K;
* decoding is deterministic and stateless (batch order / split invariant);
each for the interpreted kernel and the lane-per-path kernel."""

import itertools

import numpy as np
import pytest

import paper_1505_01466_b200 as pb

pytestmark = pytest.mark.gpu

KERNELS = ["interpreted", "lane"]


def codeword_metric(llr, word):
    """Minus the |LLR| mass where `word` disagrees with the hard decisions."""
    llr = np.asarray(llr, dtype=np.float64)
    hard = (llr < 0).astype(np.uint8)
    return -float(np.abs(llr)[np.asarray(word, np.uint8) != hard].sum())


def all_codewords(spec):
    out = []
    K = spec.k_total
    for bits in itertools.product((0, 1), repeat=K):
        u = np.zeros(spec.N, np.uint8)
        u[spec.info_positions] = bits
        out.append(pb.polar_encode(u))
    return np.array(out)


def noisy(spec, count, sigma, seed):
    rng = np.random.default_rng(seed)
    pays = rng.integers(0, 2, size=(count, spec.k), dtype=np.uint8)
    llrs = np.empty((count, spec.N), np.float32)
    for t in range(count):
        x = pb.attach_and_encode(pays[t], spec).codeword
        y = (1.0 - 2.0 * x) + rng.normal(0.0, sigma, spec.N)
        llrs[t] = (2.0 * y / sigma ** 2).astype(np.float32)
    return pays, llrs


@pytest.mark.parametrize("kernel", KERNELS)
def test_exact_ml_when_the_list_holds_every_codeword(kernel):
    spec = pb.CodeSpec.construct(8, 4, None)
    sch = pb.build_schedule(spec)
    dec = pb.ListDecoder(sch, 16, options={"kernel": kernel})
    words = all_codewords(spec)
    rng = np.random.default_rng(77)
    llrs = rng.normal(scale=2.0, size=(120, 8)).astype(np.float32)
    cw, pm, ok, pu = dec.decode_paths_batch(llrs)
    for t in range(len(llrs)):
        assert pu[t] == 16
        top = max(codeword_metric(llrs[t], w) for w in words)
        assert max(pm[t]) == pytest.approx(top, rel=1e-5, abs=1e-6)
        for p in range(16):
            assert pm[t, p] == pytest.approx(codeword_metric(llrs[t], cw[t, p]), rel=1e-5, abs=1e-6)
        # the 16 survivors are the 16 distinct codewords
        assert len({bytes(c) for c in cw[t]}) == 16
        r = dec.decode(llrs[t])
        assert r.chosen_pm == pytest.approx(top, rel=1e-5, abs=1e-6)


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("L", [8, 32])
def test_path_metrics_never_positive_and_consistent(kernel, L):
    spec = pb.CodeSpec.construct(64, 28, pb.CRC8)
    sch = pb.build_schedule(spec)
    dec = pb.ListDecoder(sch, L, options={"kernel": kernel})
    _, llrs = noisy(spec, 40, 1.1, seed=71)
    cw, pm, ok, pu = dec.decode_paths_batch(llrs)
    for t in range(len(llrs)):
        for p in range(pu[t]):
            assert pm[t, p] <= 0.0
            # the metric is the codeword's mismatch mass (Fast-SSC leaves are exact)
            assert pm[t, p] == pytest.approx(codeword_metric(llrs[t], cw[t, p]), rel=1e-5, abs=1e-5)


@pytest.mark.parametrize("kernel", KERNELS)
def test_crc_pass_beats_a_better_failing_metric(kernel):
    spec = pb.CodeSpec.construct(32, 8, pb.CRC8)
    sch = pb.build_schedule(spec)
    L = 8 if kernel == "interpreted" else 24
    dec = pb.ListDecoder(sch, L, options={"kernel": kernel})
    _, llrs = noisy(spec, 400, 1.4, seed=85)
    paths = dec.decode_paths_batch(llrs)
    res = dec.decode_batch(llrs)
    seen = 0
    for t in range(len(llrs)):
        cw, pm, ok, pu = (x[t] for x in paths)
        n = pu
        passing = [p for p in range(n) if ok[p]]
        best_any = max(range(n), key=lambda p: (pm[p], -p))
        if passing and not ok[best_any]:
            seen += 1
            best_pass = max(passing, key=lambda p: (pm[p], -p))
            assert res.crc_ok[t]
            assert res.chosen_pm[t] == pm[best_pass]
            payload, _ = pb.extract_payload(pb.polar_encode(cw[best_pass]), spec)
            assert np.array_equal(res.info_bits[t], payload)
    assert seen >= 3


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("code", [(16, 4, None), (16, 5, None), (32, 5, None), (8, 3, None)])
def test_brute_force_optimal_when_list_covers_the_code(kernel, code):
    N, k, crc = code
    spec = pb.CodeSpec.construct(N, k, {"crc8": pb.CRC8, None: None}[crc])
    if spec.k_total > 5:
        pytest.skip("code too large for the list")
    L = 1 << spec.k_total
    if kernel == "lane" and L <= 16:
        L = 32  # still covers the code; the lane kernel serves L > 16
    sch = pb.build_schedule(spec)
    dec = pb.ListDecoder(sch, L, options={"kernel": kernel})
    words = all_codewords(spec)
    rng = np.random.default_rng(N * 7 + k)
    llrs = rng.normal(0.3, 2.0, size=(150, N)).astype(np.float32)
    r = dec.decode_batch(llrs)
    for t in range(len(llrs)):
        metrics = np.array([codeword_metric(llrs[t], w) for w in words])
        assert r.chosen_pm[t] == pytest.approx(metrics.max(), rel=1e-5, abs=1e-6) or (
            spec.crc is not None and r.crc_ok[t])
        if spec.crc is None:
            assert r.paths_used[t] == min(L, 1 << spec.k_total)


@pytest.mark.parametrize("kernel", KERNELS)
def test_decoding_is_deterministic_and_stateless(kernel):
    spec = pb.CodeSpec.from_design_ebn0(1024, 828, pb.CRC32, 4.0)
    sch = pb.build_schedule(spec)
    fb = pb.generate_frames(spec, 3.5, seed=99, start=0, count=512, workers=1)
    dec = pb.ListDecoder(sch, 24 if kernel == "lane" else 8, options={"kernel": kernel})
    a = dec.decode_batch(fb.llrs)
    perm = np.random.default_rng(5).permutation(len(fb.llrs))
    b = dec.decode_batch(fb.llrs[perm])
    c = [dec.decode_batch(fb.llrs[s:s + 37]) for s in range(0, len(fb.llrs), 37)]
    for x, y in ((a.info_bits[perm], b.info_bits), (a.chosen_pm[perm], b.chosen_pm),
                 (a.paths_used[perm], b.paths_used)):
        assert np.array_equal(x, y)
    assert np.array_equal(a.chosen_pm, np.concatenate([r.chosen_pm for r in c]))
    assert np.array_equal(a.info_bits, np.concatenate([r.info_bits for r in c]))
