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
