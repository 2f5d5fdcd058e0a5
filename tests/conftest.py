import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libhcmx_gpu.so")


def _ensure_oracle():
    lib = os.path.join(ROOT, "oracle", "liboracle.so")
    src = os.path.join(ROOT, "oracle", "hcmx_oracle.c")
    if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), lib], check=True,
                       capture_output=True)


@pytest.fixture(scope="session")
def oracle():
    _ensure_oracle()
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import RefOracle
    if not RefOracle.available():
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True,
                           capture_output=True)
        else:
            pytest.skip("reference codec build (oracle/_ref) not present on this machine")
    return RefOracle()


@pytest.fixture(scope="session")
def codec_golden():
    return np.load(os.path.join(GOLDEN, "codec_golden.npz"))


@pytest.fixture(scope="session")
def hmat_golden():
    return np.load(os.path.join(GOLDEN, "hmat_golden.npz"))


@pytest.fixture(scope="session")
def gpu():
    """the product library on a real GPU -- fails (not skips) when unavailable"""
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2308_10960_b200 import _lib
    _lib.ensure_device(0)
    return _lib


def golden_cases(z):
    """yield (values, eps, scheme, e, m, scale, payload_bytes, decoded_sha256)"""
    lens = z["case_len"]
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
    vals = z["case_values"]
    pay = z["payload"]
    po = 0
    for i, r in enumerate(z["meta"]):
        c = int(r["case"])
        v = vals[starts[c]: starts[c] + lens[c]]
        n = int(r["plen"])
        yield (v, float(r["eps"]), int(r["scheme"]), int(r["e"]), int(r["m"]), float(r["scale"]),
               pay[po: po + n].tobytes(), str(z["decoded_sha256"][i]))
        po += n


def sha(values) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(values, np.float64).view(np.uint64).tobytes()).hexdigest()
