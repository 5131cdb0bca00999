"""The CPU CA oracle (oracle/ca_oracle.c) checked before it is trusted:
against golden vectors computed independently with torch float64 autograd
(tests/golden/make_golden.py) and against self-consistency properties
(split-plan composability; shared-KV gradient sums)."""
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ca_small.npz")


def golden_cases():
    z = np.load(GOLDEN)
    names = sorted({k.split("/")[0] for k in z.files})
    return {n: {k.split("/")[1]: z[k] for k in z.files if k.startswith(n + "/")} for n in names}


@pytest.mark.parametrize("name", ["whole_docs", "split_doc", "shared_kv"])
def test_oracle_matches_golden(name):
    c = golden_cases()[name]
    tasks = [tuple(t) for t in c["tasks"]]
    o, lse = oracle.ca_forward(tasks, c["q"], c["k"], c["v"])
    rows = np.concatenate([np.arange(t[0], t[0] + t[1]) for t in tasks])
    assert np.abs(o[rows] - c["o"][rows]).max() < 1e-5
    assert np.abs(lse[:, rows] - c["lse"][:, rows]).max() < 1e-5
    dq, dk, dv = oracle.ca_backward(tasks, c["q"], c["k"], c["v"], o, c["do"])
    assert np.abs(dq[rows] - c["dq"][rows]).max() < 1e-4
    assert np.abs(dk - c["dk"]).max() < 1e-4
    assert np.abs(dv - c["dv"]).max() < 1e-4


def test_split_plan_reproduces_whole_document():
    rng = np.random.default_rng(7)
    L, hq, hkv = 300, 2, 1
    q = rng.standard_normal((L, hq, 128), dtype=np.float32)
    k = rng.standard_normal((L, hkv, 128), dtype=np.float32)
    v = rng.standard_normal((L, hkv, 128), dtype=np.float32)
    do = rng.standard_normal((L, hq, 128), dtype=np.float32)
    whole = [(0, L, 0, L)]
    parts = [(0, 100, 0, 100), (100, 128, 0, 228), (228, 72, 0, 300)]
    o1, l1 = oracle.ca_forward(whole, q, k, v)
    o2, l2 = oracle.ca_forward(parts, q, k, v)
    assert np.abs(o1 - o2).max() < 1e-5 and np.abs(l1 - l2).max() < 1e-5
    g1 = oracle.ca_backward(whole, q, k, v, o1, do)
    g2 = oracle.ca_backward(parts, q, k, v, o2, do)
    for a, b in zip(g1, g2):
        assert np.abs(a - b).max() < 1e-4


def test_lse_identity():
    """LSE = log sum_j exp(s_ij) over the visible keys (natural log)."""
    rng = np.random.default_rng(3)
    q = rng.standard_normal((10, 1, 128), dtype=np.float32)
    k = rng.standard_normal((16, 1, 128), dtype=np.float32)
    v = rng.standard_normal((16, 1, 128), dtype=np.float32)
    _, lse = oracle.ca_forward([(0, 10, 0, 16)], q, k, v)
    s = (q[:, 0].astype(np.float64) @ k[:, 0].T.astype(np.float64)) / np.sqrt(128)
    for i in range(10):
        vis = s[i, : 6 + i + 1]
        assert abs(lse[0, i] - np.log(np.exp(vis).sum())) < 1e-5


def test_backward_matches_finite_differences_of_the_forward():
    """The oracle's backward is the gradient of its own forward: central
    differences of L = sum(O * G) (accumulated in fp64 from the fp32 O) with
    respect to random entries of Q, K and V, on two shards of one document
    sharing its KV prefix plus a second document, GQA group 2."""
    rng = np.random.default_rng(11)
    hq, hkv = 2, 1
    tasks = [(0, 23, 0, 23), (23, 17, 0, 40), (40, 9, 40, 9)]
    rows = 49
    q = rng.standard_normal((rows, hq, 128), dtype=np.float32)
    k = rng.standard_normal((rows, hkv, 128), dtype=np.float32)
    v = rng.standard_normal((rows, hkv, 128), dtype=np.float32)
    g = rng.standard_normal((rows, hq, 128), dtype=np.float32)

    def loss(q_, k_, v_):
        o, _ = oracle.ca_forward(tasks, q_, k_, v_)
        return float((o.astype(np.float64) * g).sum())

    o, _ = oracle.ca_forward(tasks, q, k, v)
    grads = dict(zip("qkv", oracle.ca_backward(tasks, q, k, v, o, g)))
    h = 1e-2
    worst = 0.0
    for name, x in (("q", q), ("k", k), ("v", v)):
        for _ in range(12):
            idx = tuple(int(rng.integers(0, s)) for s in x.shape)
            xp, xm = x.copy(), x.copy()
            xp[idx] += h
            xm[idx] -= h
            args_p = {"q": q, "k": k, "v": v, name: xp}
            args_m = {"q": q, "k": k, "v": v, name: xm}
            fd = (loss(args_p["q"], args_p["k"], args_p["v"]) - loss(args_m["q"], args_m["k"], args_m["v"])) / (2 * h)
            an = float(grads[name][idx])
            worst = max(worst, abs(fd - an) / (1e-1 + abs(an)))
            assert abs(fd - an) <= 3e-3 + 2e-2 * abs(an), (name, idx, fd, an)
    print("finite differences vs oracle backward, worst scaled error", worst)
