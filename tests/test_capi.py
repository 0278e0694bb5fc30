"""The C-ABI library loads and exports every entry point include/cvq.h
declares (CPU only: no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cvq.h")
SO = os.path.join(ROOT, "paper_2506_18879_b200", "libcvq_b200.so")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"CVQ_API\s+[\w\s\*]+?\b(cvq_\w+)\s*\(", src)))


def test_header_declares_the_hot_path():
    names = declared()
    for must in ("cvq_fused_attention", "cvq_encode_keys", "cvq_encoder_forward_infer",
                 "cvq_pack_key_codes", "cvq_cache_attention", "cvq_cache_decode_step",
                 "cvq_lse_combine", "cvq_cache_prefill"):
        assert must in names
    assert len(names) >= 30


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(SO):
        from paper_2506_18879_b200 import build
        build.build()
    return ctypes.CDLL(SO)


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {SO} 2>&1").read()
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, out


def test_pure_functions_need_no_gpu(lib):
    lib.cvq_predicted_flops_fused.restype = ctypes.c_uint64
    lib.cvq_predicted_flops_naive.restype = ctypes.c_uint64
    u = ctypes.c_uint64
    assert lib.cvq_predicted_flops_naive(u(8192), u(1024), u(1024)) == 17196654592
    assert lib.cvq_predicted_flops_fused(u(1), u(1), u(1), u(1), u(1)) == 5
    assert lib.cvq_predicted_flops_fused(u(0), u(1), u(1), u(1), u(1)) == 0
    assert lib.cvq_abi_version() == 1


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="GPU present")
def test_context_fails_loudly_without_gpu(lib):
    h = ctypes.c_void_p()
    rc = lib.cvq_context_create(0, None, ctypes.byref(h))
    assert rc in (1, 5)  # EINVAL (no device) or ECUDA: never a silent CPU path
    lib.cvq_last_error.restype = ctypes.c_char_p
    assert lib.cvq_last_error()
