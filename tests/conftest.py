import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsaloba.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    import build_native

    build_native.build_synth()
    build_native.build_oracle()


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def load_tsv(name):
    rows = []
    with open(os.path.join(ROOT, "tests", "golden", name)) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            c = line.rstrip("\n").split("\t")
            rows.append(dict(mode=c[0], q=c[1], t=c[2], match=int(c[3]), mismatch=int(c[4]), alpha=int(c[5]),
                             beta=int(c[6]), h0=int(c[7]), expect=(int(c[8]), int(c[9]), int(c[10])),
                             note=c[11] if len(c) > 11 else ""))
    return rows
