"""The exact sliding oracle on the GPU: ExactSlidingOracle
(exact_oracle.hpp:25-62, exact_oracle.cpp:22-101). Windows (cadence, exact
per-host distinct-peer counts >= theta, order) must be byte-identical with the
reference's own exact_detect; the max_pairs budget fails like the reference;
score() (exact_oracle.cpp:105-132) rates the sketch detection against it."""
import numpy as np
import pytest

from paper_1805_09246_b200 import abi, synth


def exact_restated(pairs, off, theta, k):
    """plain restatement: a pair is live in the window ending at slice s iff
    its last sighting is in (s - k, s]; a window per completed slice from k-1
    on (every slice but the last) plus the partial one at stream end"""
    last = {}
    out = []
    n = len(off) - 1
    for s in range(n):
        for i in range(int(off[s]), int(off[s + 1])):
            last[(int(pairs["aip"][i]), int(pairs["bip"][i]))] = s
        partial = s == n - 1
        if s + 1 >= k or partial:
            counts = {}
            for (a, _), t in last.items():
                if t > s - k:
                    counts[a] = counts.get(a, 0) + 1
            sup = sorted(((a, c) for a, c in counts.items() if c >= theta),
                         key=lambda x: (-x[1], x[0]))
            out.append((s, partial, sup))
    return out


def small_trace(seed=5, slices=12, per_slice=4000, hosts=30):
    rng = np.random.default_rng(seed)
    pairs = np.zeros(slices * per_slice, dtype=abi.PAIR_DTYPE)
    pairs["aip"] = 0x0A000000 + rng.integers(0, hosts, len(pairs))
    pairs["bip"] = rng.integers(0, 3000, len(pairs)).astype(np.uint32) * 7919
    off = np.arange(slices + 1, dtype=np.uint64) * per_slice
    return pairs, off


def test_restatement_matches_reference(ref):
    pairs, off = small_trace()
    got = exact_restated(pairs, off, theta=100, k=4)
    exp = abi.parse_truth(ref.exact_detect(pairs, off, 100, 4))
    assert got == exp


def test_score_restatement():
    truth = [(1, 500), (2, 400), (3, 300)]
    s = abi.score([1, 2, 9], truth)
    assert (s["fp"], s["fn"], s["n_true"]) == (1, 1, 3)
    assert abs(s["tfr"] - 2 / 3) < 1e-12 and s["defined"]
    assert not abi.score([4], [])["defined"]


@pytest.mark.gpu
@pytest.mark.parametrize("k,theta", [(4, 100), (1, 50), (12, 300)])
def test_gpu_exact_small_vs_reference(ref, k, theta):
    from paper_1805_09246_b200 import native

    pairs, off = small_trace()
    o = native.ExactOracle(theta=theta, k=k, max_pairs=1 << 20)
    o.process_slices(pairs, off)
    o.finish()
    assert o.take_windows() == ref.exact_detect(pairs, off, theta, k)


@pytest.mark.gpu
def test_gpu_exact_c2_scaled_vs_reference_and_scores_detection(ref):
    """a 3M-packet C2-shaped trace: identical truth windows, and the sketch
    detection scored against them (the planted super points are found)"""
    import torch

    from paper_1805_09246_b200 import native

    w = synth.scaled(synth.WORKLOADS["c2"], packets=3_000_000, n_slices=30, planted=30,
                     planted_spread=10)
    pairs, off = synth.trace(w).generate()
    k, theta = 10, 1024
    d = torch.from_numpy(pairs.view(np.uint8)).cuda()
    o = native.ExactOracle(theta=theta, k=k, max_pairs=1 << 23)
    o.process_slices(offsets=off, device_ptr=d.data_ptr())
    o.finish()
    blob = o.take_windows()
    assert blob == ref.exact_detect(pairs, off, theta, k)
    truth = abi.parse_truth(blob)
    e = native.WindowEngine.from_params(w.sketch_params(), w.window_config(k=k, t0_us=0))
    e.process_slices(pairs, off)
    e.finish()
    reps = abi.parse_blobs(e.take_reports())
    assert [r.window_end_slice for r in reps] == [t[0] for t in truth]
    fnr = [abi.score([a for a, _, _ in r.entries], t[2])["fnr"] for r, t in zip(reps, truth)
           if t[2]]
    assert fnr and max(fnr) <= 0.2


@pytest.mark.gpu
def test_gpu_exact_pair_budget():
    from paper_1805_09246_b200 import native

    pairs, off = small_trace()
    o = native.ExactOracle(theta=100, k=4, max_pairs=1000)
    with pytest.raises(abi.ResourceError, match="distinct pair budget"):
        o.process_slices(pairs, off)
    with pytest.raises(abi.ConfigError):
        native.ExactOracle(k=0)
