import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


# Forward-path selector for the parity tests: "fused" forces the fused
# recurrent+parallel kernel (K12, L = 128) even below one wave of chains,
# "split" forces the K1 state scan + K2 parallel kernel pair.
FWD_PATHS = {"fused": ("TFLA_FORCE_FUSED_FWD", "TFLA_NO_FUSED_FWD"),
             "split": ("TFLA_NO_FUSED_FWD", "TFLA_FORCE_FUSED_FWD")}


@pytest.fixture(params=sorted(FWD_PATHS))
def fwd_path(request, monkeypatch):
    on, off = FWD_PATHS[request.param]
    monkeypatch.setenv(on, "1")
    monkeypatch.delenv(off, raising=False)
    return request.param
