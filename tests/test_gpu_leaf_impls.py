"""The TSQR leaf kernel and the Jacobi SVD have several paths (warp-specialised default, CTA-wide,
explicit-panel fallback forced, warp roles assigned without %warpid) selected by
environment variables that the library reads once per process; each is checked in a
subprocess against the same parity tests."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"JQ_TSQR_IMPL": "cta"}, {"JQ_TSQR_EXPLICIT": "1"},
                                 {"JQ_TSQR_IMPL": "cta", "JQ_TSQR_EXPLICIT": "1"},
                                 {"JQ_TSQR_DEBUG": "8"}, {"JQ_TSQR_CHAIN": "householder"},
                                 {"JQ_TSQR_CHAIN": "householder", "JQ_TSQR_IMPL": "cta"},
                                 {"JQ_TSQR_REDUCERS": "1"}, {"JQ_TSQR_WS128": "kw16"}, {"JQ_TSQR_WS128": "kw24"},
                                 {"JQ_TSQR_WS32": "kw32"}, {"JQ_TSQR_WS64": "staged"}, {"JQ_TSQR_WS64": "w8"},
                                 {"JQ_TSQR_WS64": "staged", "JQ_TSQR_CHAIN": "householder"},
                                 {"JQ_TSQR_STAGED": "1"}, {"JQ_TSQR_STAGED": "1", "JQ_TSQR_IMPL": "cta"}],
                         ids=["cta", "ws-explicit", "cta-explicit", "ws-fixed-roles", "ws-reflector-chain",
                              "cta-reflector-chain", "ws-reducer-warps", "ws-np128-kw16", "ws-np128-kw24", "ws-np32-kw32", "ws-np64-staged", "ws-np64-w8", "ws-np64-staged-reflector",
                              "staged-tree", "cta-staged"])
def test_leaf_impl_parity(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", "figaro or householder or shard"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_svd_v_overlap_parity():
    # JQ_SVD_V_OVERLAP=1: the V replay concurrently with the sweeps (opt-in)
    e = dict(os.environ, JQ_SVD_V_OVERLAP="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", "svd"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_svd_coop_impl_parity():
    # JQ_SVD_IMPL=coop: the grid-barrier Jacobi kernel instead of the cluster kernel
    e = dict(os.environ, JQ_SVD_IMPL="coop")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", "svd"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_svd_v_one_warp_replay_parity():
    # JQ_SVD_V1=1: the one-warp-per-row V replay instead of the four-warp default
    e = dict(os.environ, JQ_SVD_V1="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", "svd"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_segscan_narrow_pass_parity():
    # JQ_SEGSCAN_TINY=0: keyed <= 16-column tile passes on the one-row-per-load narrow kernel
    e = dict(os.environ, JQ_SEGSCAN_TINY="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", "figaro or head_tail or reduce"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_svd_generic_cluster_kernel_parity():
    # JQ_SVD_GENERIC=1: the runtime-np cluster kernel also at np = 256
    e = dict(os.environ, JQ_SVD_GENERIC="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", "svd"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_footnote_serial_trees_parity():
    # JQ_FOOTNOTE_SERIAL_TREES=1: the keyed footnote's side trees on the main stream
    e = dict(os.environ, JQ_FOOTNOTE_SERIAL_TREES="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", "figaro"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
