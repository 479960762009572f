"""CPU-side checks of the C ABI: the library builds/loads and exports every symbol that
include/efunc.h declares; struct layouts of the binding match the header. No GPU calls."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "efunc.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"EFUNC_API\s+[\w\s\*]+?\b(efunc_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2505_21319_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_north_star_entry_points():
    syms = declared_symbols()
    for name in ["efunc_create", "efunc_forward", "efunc_backward", "efunc_adamw_step", "efunc_eval_grad"]:
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (efunc_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_binding_covers_every_symbol():
    from paper_2505_21319_b200 import efunc
    assert sorted(efunc.EXPORTED) == declared_symbols()


def test_abi_version_callable_without_gpu(lib):
    lib.efunc_abi_version.restype = ctypes.c_int32
    assert lib.efunc_abi_version() == 1


def test_variant_channel_counts_without_gpu(lib):
    """efunc_channels (NEXT-4) against Table 3's "Ch" column and the variant
    oracle's layout."""
    from oracle import variant_oracle as vo
    lib.efunc_channels.restype = ctypes.c_int32
    lib.efunc_channels.argtypes = [ctypes.c_int32, ctypes.c_int32]
    assert lib.efunc_channels(0, 1) == 13 and lib.efunc_channels(0, 0) == 13  # Full-4 / G-0 tie
    assert lib.efunc_channels(1, 2) == 11   # G-7
    assert lib.efunc_channels(1, 1) == 5    # G-6
    assert lib.efunc_channels(1, 0) == 2    # G-5
    assert lib.efunc_channels(2, 1) == 8    # Full-1
    for v, banks in ((0, vo.BOTH), (1, vo.GRID), (2, vo.OFFSET)):
        assert lib.efunc_channels(v, 2) == vo.n_channels(banks, 2)
    assert lib.efunc_channels(3, 1) == -1 and lib.efunc_channels(0, 3) == -1


def test_struct_sizes_match_header():
    """Compile a tiny C program against the header and compare sizeof with the ctypes mirrors."""
    from paper_2505_21319_b200 import efunc
    src = r'''
    #include <stdio.h>
    #include "efunc.h"
    int main(){printf("%zu %zu %zu %zu\n", sizeof(efunc_config), sizeof(efunc_loss),
                       sizeof(efunc_adamw), sizeof(efunc_stats)); return 0;}
    '''
    tmp = "/tmp/efunc_sizeof"
    with open(tmp + ".c", "w") as fh:
        fh.write(src)
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), tmp + ".c", "-o", tmp], check=True)
    sizes = [int(x) for x in subprocess.run([tmp], capture_output=True, text=True).stdout.split()]
    assert sizes == [ctypes.sizeof(efunc.Config), ctypes.sizeof(efunc.Loss),
                     ctypes.sizeof(efunc.AdamWParams), ctypes.sizeof(efunc.Stats)]


def test_create_fails_cleanly_without_gpu(lib):
    """Without a device the ABI returns an error code (never crashes / throws)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2505_21319_b200 import efunc
    L = efunc.load_library()
    cfg = efunc.Config(8, 1, 0, 20.0, 0, 0, 0)
    h = ctypes.c_void_p()
    st = L.efunc_create(ctypes.byref(cfg), None, ctypes.byref(h))
    assert st in (efunc.ECUDA, efunc.EINVAL)
    assert L.efunc_last_error(None)


def test_default_decay_mask_covers_polynomial_coefficients_only():
    """The binding's default AdamW decay mask (reading R-10, SPEC D15) decays the polynomial
    coefficients c, g (and H) of every bank of a layout and never the scales s or offsets Delta."""
    from oracle import variant_oracle as vo
    from paper_2505_21319_b200 import efunc
    for variant, banks in ((efunc.VARIANT_GRID, vo.GRID), (efunc.VARIANT_OFFSET, vo.OFFSET),
                           (efunc.VARIANT_COMBINED, vo.BOTH)):
        for degree in (0, 1, 2):
            lay = vo.layout(banks, degree)
            want = 0
            for key in ("grid", "off"):
                if lay[key] is not None:
                    for c in range(1, 1 + vo.NCOEF[degree]):
                        want |= 1 << (lay[key] + c)
            got = efunc._coef_mask(variant, degree)
            if variant == efunc.VARIANT_COMBINED and degree == 0:
                assert got == efunc.DEFAULT_DECAY_MASK  # the 13-channel tie keeps its mask
            else:
                assert got == want, (variant, degree, bin(got), bin(want))
