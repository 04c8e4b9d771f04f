"""CPU-side checks of the C-ABI library (-m "not gpu"): it builds, loads,
exports every symbol include/casc.h declares, and its host-only logic
(widths, sizes, argument validation) behaves as documented.  No compute call
is made without a GPU."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "casc.h")


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as ge
    ge.build_cuda()
    from paper_2303_04353_b200 import _lib
    return _lib


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(casc_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_expected_entry_points():
    names = declared_functions()
    for must in ("casc_gemm_fp64x2", "casc_split_a", "casc_split_b", "casc_debug_bins",
                 "casc_gemm_packed", "casc_status_string", "casc_workspace_bytes"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    import paper_2303_04353_b200 as casc
    so = casc.LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (casc_[a-z0-9_]+)", out))
    for name in declared_functions():
        assert name in exported, name
        assert hasattr(lib, name)
        assert name in casc.EXPORTED


def test_library_is_sm100a_only(lib):
    import paper_2303_04353_b200 as casc
    out = subprocess.run(["cuobjdump", "--list-elf", casc.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", casc.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "DMMA.8x8x4" in sass      # FP64 tensor-core MMA in the fused kernel
    assert "UBLKCP" in sass          # TMA bulk copies
    assert "LDTM" in sass and "STTM" in sass  # tensor-memory C accumulator
    # the product kernel (no debug export, no alpha/beta) and the split kernels
    # are spill-free
    funcs = re.split(r"\n\s*Function : ", sass)
    main = [f for f in funcs if f.startswith("_ZN4casc16casc_gemm_kernelILb0ELb0ELb0ELb0ELb0E")]
    splits = [f for f in funcs if "split_a_kernel" in f[:60] or "split_b_kernel" in f[:60]]
    assert len(main) == 1 and len(splits) == 4
    for f in main + splits:
        assert "LDL" not in f and "STL" not in f


def test_widths_and_sizes(lib):
    import paper_2303_04353_b200 as casc
    assert casc.casc_select_widths(256) == (22, 21, 21)
    assert casc.casc_select_widths(64) == (23, 22, 22)
    assert casc.casc_select_widths(16384) == (22, 21, 21)
    assert casc.casc_select_widths(1) == (26, 25, 25)
    kb = casc.casc_packed_b_block_bytes(300)
    assert casc.casc_packed_b_bytes(300, 130) == 3 * kb
    assert casc.casc_packed_a_bytes(65, 300) == 2 * casc.casc_packed_a_block_bytes(300)
    # k = 300 -> kpad 304 -> 76 k4-steps; 2 panels of exponents
    assert casc.casc_packed_a_block_bytes(300) == 76 * 1024 * 8 + 2 * 64 * 4
    assert casc.casc_packed_b_block_bytes(300) == 76 * 1792 * 8 + 2 * 64 * 4
    # + the fused kernel's 256-byte scratch head (wave counter, WIDE list count)
    assert casc.casc_workspace_bytes(0, 5, 5) == casc.casc_packed_b_bytes(5, 5) + 256
    assert casc.casc_status_string(0) == "CASC_OK"
    assert "invalid" in casc.casc_status_string(1)


def test_invalid_arguments_rejected_before_any_cuda_call(lib):
    P = ctypes.c_void_p
    fake = P(0x1000)
    call = lambda m, n, k, lda, ldb, ldc, a=fake, c=P(0x900000): lib.casc_gemm_fp64x2(
        m, n, k, a, a, lda, fake, fake, ldb, c, P(0xA00000), ldc, None, None)
    assert call(-1, 4, 4, 4, 4, 4) == 1
    assert call(4, 4, 4, 3, 4, 4) == 1          # lda < k
    assert call(4, 4, 4, 4, 3, 4) == 1          # ldb < n
    assert call(4, 4, 4, 4, 4, 3) == 1          # ldc < n
    assert call(4, 4, 4, 4, 4, 4, a=None) == 1  # NULL with non-zero size
    # C overlapping A
    assert lib.casc_gemm_fp64x2(4, 4, 4, fake, P(0x9000), 4, P(0x20000), P(0x30000), 4,
                                P(0x1008), P(0x40000), 4, None, None) == 1
    assert lib.casc_select_widths(-1, (ctypes.c_int * 3)()) == 1
    assert lib.casc_debug_bins(4, 4, 4, fake, fake, 4, fake, fake, 4, 1, P(0x5000), None) == 1
