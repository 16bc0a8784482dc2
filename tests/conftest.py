import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU; run with -m gpu")
    config.addinivalue_line("markers", "slow: larger CPU oracle cases")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import REF_SO, RefLib

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def ctx():
    """GPU context; GPU tests FAIL (not skip) when the CUDA path cannot run."""
    from paper_2203_08498_b200 import api

    return api.Context(0)


@pytest.fixture(scope="session")
def problems():
    from paper_2203_08498_b200 import problems as P

    return P


def laplacian_2d(grid: int):
    """gen_laplacian_2d (src/csr_matrix.cpp:124-144) restated for fixtures: 5-point, diag 4."""
    n = grid * grid
    rs, ci, va = [0], [], []
    for y in range(grid):
        for x in range(grid):
            p = y * grid + x
            if y > 0:
                ci.append(p - grid), va.append(-1.0)
            if x > 0:
                ci.append(p - 1), va.append(-1.0)
            ci.append(p), va.append(4.0)
            if x < grid - 1:
                ci.append(p + 1), va.append(-1.0)
            if y < grid - 1:
                ci.append(p + grid), va.append(-1.0)
            rs.append(len(ci))
    return n, np.array(rs, np.int32), np.array(ci, np.int32), np.array(va)


def random_sdd_spd(n: int, density: float, seed: int, oracle_obj):
    """testsup::random_sdd_spd (tests/test_support.hpp:73-102) restated: symmetric pattern,
    values U[-1,1), diagonal = |row| sum + 1 + U[0,1); same UniformPm1 draw order."""
    # one UniformPm1 stream: one draw per (i < j) pair, one more when the pair is kept, then
    # one per diagonal -- the fixture's draw order
    total_needed = n * n * 2 + n
    stream = oracle_obj.uniform_pm1(seed, 0, total_needed)
    pos = 0
    rows = [dict() for _ in range(n)]
    for i in range(n):
        for j in range(i + 1, n):
            u01 = 0.5 * (stream[pos] + 1.0)
            pos += 1
            if u01 < density:
                v = stream[pos]
                pos += 1
                rows[i][j] = v
                rows[j][i] = v
    for i in range(n):
        s = sum(abs(v) for v in rows[i].values())
        rows[i][i] = s + 1.0 + 0.5 * (stream[pos] + 1.0)
        pos += 1
    rs, ci, va = [0], [], []
    for i in range(n):
        for j in sorted(rows[i]):
            ci.append(j)
            va.append(rows[i][j])
        rs.append(len(ci))
    return n, np.array(rs, np.int32), np.array(ci, np.int32), np.array(va)


def spectral_fixture(n, smalls, seed, oracle_obj):
    """testsup::make_spectral_fixture (tests/test_support.hpp:27-68) restated: A = Q diag(l) Q^T,
    Q = MGS of seeded uniform columns, l = smalls then 1 + 0.5 U[-1,1); dense CSR."""
    stream = oracle_obj.uniform_pm1(seed, 0, n * n + n)
    raw = stream[: n * n].reshape(n, n)
    q = oracle_obj.mgs(raw, 1e-12)
    assert q.shape[0] == n
    lam = list(smalls)
    pos = n * n
    while len(lam) < n:
        lam.append(1.0 + 0.5 * stream[pos])
        pos += 1
    dense = np.zeros((n, n))
    for k in range(n):
        f = lam[k] * q[k]
        for i in range(n):
            dense[i, i:] += f[i] * q[k, i:]
    full = np.triu(dense) + np.triu(dense, 1).T
    rs = np.arange(0, n * n + 1, n, dtype=np.int32)
    ci = np.tile(np.arange(n, dtype=np.int32), n)
    return n, rs, ci, full.reshape(-1).copy(), np.array(lam), q


@pytest.fixture(scope="session")
def parity_log():
    """Record the achieved difference and the bar of a parity check (gpurun_out/parity/*.jsonl;
    the round's copy is committed as profiles/parity_r2.json), so a green test also shows how far
    from its bar it passed."""
    import json

    d = os.path.join(ROOT, "gpurun_out", "parity")
    os.makedirs(d, exist_ok=True)
    path = os.path.join(d, f"parity_{os.getpid()}.jsonl")

    def log(test: str, **kw):
        with open(path, "a") as f:
            f.write(json.dumps({"test": test, **{k: (float(v) if isinstance(v, (np.floating, float)) else v)
                                                 for k, v in kw.items()}}, default=str) + "\n")

    return log
