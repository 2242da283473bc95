"""The A-distribution studies (studies/a_distribution.py, PAPER.md Sec.
4.1-4.2) on a reduced grid: the paper's qualitative statements about Figs.
5-6 hold for the advanced codec (the oracle), and, on a GPU, the CUDA
codecs' streams of the study are the oracle's."""
import numpy as np
import pytest

from studies import a_distribution as S


@pytest.fixture(scope="module")
def res():
    return S.run(trials=6, N=10000, gpu=None, block_sizes=[30, 154, 300, 10000], signal_counts=[4, 500, 1000])


def adv(res, d, L):
    return res["block_size_sweep"][d][str(L)]["advanced_core"]


def test_blocking_beats_the_whole_vector(res):
    # PAPER.md:344 "blocks of 154 elements ... larger than 17 % to the basic compression"
    p = res["paper_pair_1855"]
    assert p["L154"]["advanced_core"] > 1.10 * p["whole"]["advanced_core"]
    assert abs(p["whole"]["advanced_core"] / 2.10361 - 1) < 0.03
    assert abs(p["L154"]["advanced_core"] / 2.47054 - 1) < 0.04


def test_noise_spread_and_signal_range(res):
    # sigma has a high influence, the signal range a lighter one
    best = max([154, 300], key=lambda L: adv(res, "s500_r45k", L))
    assert adv(res, "s500_r45k", best) > adv(res, "s1000_r45k", best) * 1.05
    for L in (154, 300, 10000):
        assert adv(res, "s500_r100k", L) <= adv(res, "s500_r45k", L)
    assert adv(res, "s500_r100k", best) > 0.95 * adv(res, "s500_r45k", best)


def test_too_long_blocks_lose(res):
    # "The compression ratio is weaker if the blocks are too long"
    for d in S.DISTS:
        assert adv(res, d, 10000) < 0.9 * max(adv(res, d, 154), adv(res, d, 300))
    assert adv(res, "s500_r45k", 30) < adv(res, "s500_r45k", 154)  # and if too short


def test_signal_fraction_plateau(res):
    # PAPER.md:378 "The compression ratio is constant from 10 %"
    for d in S.DISTS:
        r = res["signal_sweep"][d]
        assert abs(r["1000"]["advanced_core"] / r["500"]["advanced_core"] - 1) < 0.03
        assert r["4"]["advanced_core"] > r["500"]["advanced_core"]


@pytest.mark.gpu
def test_gpu_codecs_in_the_study():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1805_01844_b200 import polycomp as pc
    pc.poly_init()
    r = S.run(trials=3, N=4000, gpu=(torch, pc), block_sizes=[30, 154, 4000], signal_counts=[4, 400])
    for sweep in (r["block_size_sweep"], r["signal_sweep"]):
        for d, row in sweep.items():
            if d == "block_len":
                continue
            for p in row.values():
                assert p["gpu_basic_bit_exact"]
                if "gpu_advanced_bit_exact" in p:
                    assert p["gpu_advanced_bit_exact"]
