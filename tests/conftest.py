import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100) device")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


@pytest.fixture(scope="session")
def ctx():
    import paper_1711_00289_b200 as P
    c = P.Context(0)
    yield c
    c.close()


def env_context(**env):
    """A Context created with CVG_* tuning switches set (they are read at
    context creation), e.g. env_context(CVG_STRICT="1")."""
    import paper_1711_00289_b200 as P
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return P.Context(0)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


def exp_arguments(n=1_000_000, seed=3):
    """Arguments for the exp pinning tests: the Newton range of the deep
    solves (x = 0.05 t, t from the guesses down to far-left roots), the
    shallow exp(-50 q) range, the scaled special cases |x| in [512, 1024),
    tiny |x| < 2^-54, non-finite values and random bit patterns."""
    import numpy as np
    r = np.random.default_rng(seed)
    t = r.uniform(-6100.0, 1300.0, n)
    parts = [0.05 * t, r.uniform(-760.0, 720.0, n // 2), -50.0 * r.uniform(0.0, 0.03, n // 4),
             r.uniform(-1.0, 1.0, n // 8) * 2.0 ** -r.integers(40, 80, n // 8),
             r.integers(0, 2 ** 63, n // 8, dtype=np.int64).view(np.float64),
             np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 709.78, 709.79, -708.4, -745.1, -745.2, 512.0,
                       -512.0, 1024.0, -1024.0, 2.0 ** -54, -(2.0 ** -54), 2.0 ** -55])]
    return np.concatenate(parts)
