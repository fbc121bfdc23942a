"""Test configuration.

* ``-m gpu`` tests need a B200 and call the CUDA path through the C ABI.
* everything else runs on CPU: the oracle against golden vectors, the
  product's kinetics compiled for the host, the ABI export table, and the
  multi-slab host logic over gloo.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

NATIVE = os.path.join(ROOT, "tests", "native")
KIN_SO = os.path.join(NATIVE, "_build", "libkinetics_host.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def _newer(target, *sources):
    return os.path.exists(target) and all(os.path.getmtime(s) <= os.path.getmtime(target) for s in sources)


def build_kinetics_host():
    """Compile the product's __host__ __device__ kinetics for the CPU."""
    src = os.path.join(NATIVE, "kinetics_host.cpp")
    hdr = os.path.join(ROOT, "paper_2202_13821_b200", "csrc", "hgks_kinetics.cuh")
    if _newer(KIN_SO, src, hdr):
        return KIN_SO
    os.makedirs(os.path.dirname(KIN_SO), exist_ok=True)
    cuda_inc = "/usr/local/cuda/include"
    cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-I", cuda_inc,
           "-I", os.path.dirname(hdr), "-x", "c++", src, "-o", KIN_SO]
    subprocess.run(cmd, check=True)
    return KIN_SO


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build(ref=True)
    return oracle


@pytest.fixture(scope="session")
def kin_host():
    import ctypes
    return ctypes.CDLL(build_kinetics_host())


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


@pytest.fixture(scope="session")
def hgks():
    if not _has_gpu():
        pytest.skip("no CUDA device")
    from paper_2202_13821_b200 import build as B
    B.build()
    import paper_2202_13821_b200 as P
    return P
