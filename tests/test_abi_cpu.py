"""CPU-only checks of the C-ABI library: it loads, exports every function
include/wally.h declares, and its host-only entry points behave (no GPU
compute is called here)."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in sorted(os.listdir(os.path.join(ROOT, "include"))):
        if h.endswith(".h"):
            src = open(os.path.join(ROOT, "include", h)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names |= set(re.findall(r"\b(wally_[a-z_0-9]+)\s*\(", src))
    return sorted(names)


@pytest.fixture(scope="module")
def wl():
    from paper_2406_06761_b200 import build
    build.build()
    from paper_2406_06761_b200 import wally
    return wally


def test_library_exports_every_declared_symbol(wl):
    names = declared_functions()
    assert len(names) >= 15
    so = ctypes.CDLL(wl._LIB_PATH)
    for n in names:
        assert hasattr(so, n), n
    from paper_2406_06761_b200 import simd
    assert sorted(wl.EXPORTED + simd.EXPORTED) == names


def test_library_is_sm100a_only(wl):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", wl._LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("n,L", [(4096, 2), (4096, 3), (8192, 4), (1024, 1), (2048, 4)])
def test_find_moduli_agrees_with_oracle(wl, n, L):
    assert wl.wally_find_moduli(n, L) == capi.find_primes(n, L)


def test_find_moduli_rejects_bad_args(wl):
    with pytest.raises(wl.WallyError):
        wl.wally_find_moduli(1000, 2)
    with pytest.raises(wl.WallyError):
        wl.wally_find_moduli(4096, 5)


def test_create_validates_params_before_touching_the_device(wl):
    p = wl.wally_params(n=4096, num_limbs=2, t=65537, d=128)
    for i, q in enumerate(wl.wally_find_moduli(4096, 2)):
        p.moduli[i] = q
    h = ctypes.c_void_p()
    bad = wl.wally_params(n=3000, num_limbs=2, t=65537, d=128)
    assert wl.lib.wally_create(ctypes.byref(bad), 0, ctypes.byref(h)) == -2
    bad = wl.wally_params(n=4096, num_limbs=2, t=65537, d=128)
    bad.moduli[0], bad.moduli[1] = 1073668097, 1073668097 + 8192  # not prime / not ascending-prime
    assert wl.lib.wally_create(ctypes.byref(bad), 0, ctypes.byref(h)) == -2
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert wl.lib.wally_create(ctypes.byref(p), 0, ctypes.byref(h)) == -6
        assert b"CUDA" in wl.lib.wally_last_error(None) or b"device" in wl.lib.wally_last_error(None)


def test_simd_default_moduli_and_param_validation(wl):
    """Host-only parts of include/wally_simd.h: the default moduli (reading S25: the coefficient path's L
    limbs, then the next NTT-friendly prime below them) and parameter validation before any device work."""
    from paper_2406_06761_b200 import simd
    for n, L in [(4096, 3), (4096, 2), (8192, 4), (1024, 1)]:
        m = simd.simd_moduli(n, L)
        assert m[:L] == wl.wally_find_moduli(n, L)
        allp = capi.find_primes(n, L + 1)
        assert m[L] == allp[0] and m[L] < m[0]
    bad = [
        dict(n=3000, L=2, d=16),                      # n not supported
        dict(n=4096, L=2, d=4096),                    # d > n/2
        dict(n=4096, L=2, d=16, t=65539),             # t not = 1 mod 2n (and not prime)
        dict(n=4096, L=2, d=16, swap=True),           # special prime above q_0
        dict(n=4096, L=2, d=16, baby=17),             # g > d
    ]
    for b in bad:
        n, L = b["n"], b["L"]
        p = simd.wally_simd_params(n=n, num_limbs=L, t=b.get("t", 65537), d=b["d"], baby=b.get("baby", 0))
        mods = simd.simd_moduli(4096, L) if n == 3000 else simd.simd_moduli(n, L)
        if b.get("swap"):
            mods = [mods[L]] + mods[1:L] + [mods[0]]
        for i, q in enumerate(mods):
            p.moduli[i] = q
        h = ctypes.c_void_p()
        rc = wl.lib.wally_simd_create(ctypes.byref(p), 0, ctypes.byref(h))
        assert rc == -2, (b, rc)
        assert wl.lib.wally_simd_last_error(None)
