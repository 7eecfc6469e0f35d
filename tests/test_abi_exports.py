"""CPU checks of the C-ABI library: it loads, exports every symbol include/sphinx.h
declares, and rejects invalid host-visible arguments before touching a GPU."""
import ctypes
import os
import re

import pytest

import paper_2511_18672_b200 as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    hdr = open(os.path.join(ROOT, "include", "sphinx.h")).read()
    return sorted(set(re.findall(r"SPHINX_API\s+[\w\s\*]+?\b(sphinx_\w+)\s*\(", hdr)))


def test_header_and_binding_agree():
    assert _declared() == sorted(sp.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = sp.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.sphinx_abi_version() == sp.ABI_VERSION


def test_invalid_arguments_rejected_on_host():
    lib = sp.load()
    null = None
    # n = 0 (S:44 invalid-argument), before any device query
    assert lib.sphinx_compact_blocks(null, 0, 9, 9, null, 0, 0, null, null, null) == sp.ERR_INVALID_ARGUMENT
    assert lib.sphinx_compact_blocks(null, 1, 9, 9, null, 0, 0, ctypes.c_void_p(16),
                                     ctypes.c_void_p(16), null) == sp.ERR_INVALID_ARGUMENT  # ACTIVE needs mask
    assert lib.sphinx_noise_inject(null, null, null, 1, 8, 8, 4, 8, null, null, 1, null, null, 50,
                                   null) == sp.ERR_INVALID_ARGUMENT
    # tau_o outside [0,1]
    masks = (ctypes.c_void_p * 1)(16)
    assert lib.sphinx_block_mask(ctypes.c_void_p(16), null, null, 1.5, 1, 16, 16, 1, 4, 1,
                                 ctypes.cast(masks, ctypes.c_void_p), null, null, null,
                                 null) == sp.ERR_INVALID_ARGUMENT
    # channels not a multiple of 8 -> unsupported (no fallback)
    p = ctypes.c_void_p(1024)
    assert lib.sphinx_sparse_conv3x3(p, p, null, p, sp.F32, 1, 16, 16, 12, 32, 4, p, p, 16, null, 0,
                                     null) == sp.ERR_UNSUPPORTED
    # workspace: split-K counters + edge plan (capacity ids) + partial tiles; grows with N
    small = lib.sphinx_conv_workspace_size(1, 16, 16, 32, 32, 4)
    big = lib.sphinx_conv_workspace_size(168, 16, 16, 32, 32, 4)
    assert small > 4096 and big - small >= (168 - 1) * 16 * 4 - 256
    assert lib.sphinx_conv_workspace_size(0, 16, 16, 32, 32, 4) == 0
    # _ex: flags outside REUSE_PLAN | LIST_READY | INPUT_READY are rejected before any device query
    assert (sp.CONV_REUSE_PLAN, sp.CONV_LIST_READY, sp.CONV_INPUT_READY) == (1, 2, 4)
    assert lib.sphinx_sparse_conv3x3_ex(p, p, null, null, p, sp.BF16, 1, 16, 16, 32, 32, 4, p, p, 16, p,
                                        1 << 20, 8, null) == sp.ERR_INVALID_ARGUMENT


def test_next3_host_validation():
    """NEXT-3 entry points reject bad host-visible arguments before touching a GPU."""
    lib = sp.load()
    p, null = ctypes.c_void_p(1024), None
    # c % groups != 0 -> invalid; c % 8 != 0 -> unsupported
    assert lib.sphinx_gn_block_stats(p, 1, 16, 16, 40, 32, 8, p, p, 4, p, null) == sp.ERR_INVALID_ARGUMENT
    assert lib.sphinx_gn_block_stats(p, 1, 16, 16, 36, 4, 8, p, p, 4, p, null) == sp.ERR_UNSUPPORTED
    assert lib.sphinx_gn_silu(p, p, p, p, 1e-6, 1, 16, 16, 32, 8, 8, p, p, 4, p, null) == \
        sp.ERR_INVALID_ARGUMENT  # a aliases x
    assert lib.sphinx_gn_stats_size(2, 18, 18, 32, 8) == 2 * 9 * 32 * 8 + 2 * 32 * 8
    assert lib.sphinx_sparse_conv3x3_residual(p, p, null, null, p, sp.F32, 1, 16, 16, 32, 32, 8, p, p,
                                              4, null, 0, null) == sp.ERR_INVALID_ARGUMENT
    q = ctypes.c_void_p(2048)
    # h_buf aliases x
    assert lib.sphinx_sparse_resblock(p, p, null, p, null, p, p, p, p, 32, 1e-6, p, q, ctypes.c_void_p(4096),
                                      q, sp.BF16, ctypes.c_void_p(8192), 1, 16, 16, 64, 8, p, p, 4, null,
                                      0, null) == sp.ERR_INVALID_ARGUMENT


def test_next4_host_validation():
    lib = sp.load()
    p, null = ctypes.c_void_p(1024), None
    q = ctypes.c_void_p(4096)
    # head dim must be 64 (c / heads), frames_per_seq must divide N
    assert lib.sphinx_temporal_attention(p, q, 4, 8, 8, 128, 1, 2, 8, p, p, 4, p, 64, null) == sp.ERR_UNSUPPORTED
    assert lib.sphinx_temporal_attention(p, q, 5, 8, 8, 128, 2, 2, 8, p, p, 5, p, 64, null) == \
        sp.ERR_INVALID_ARGUMENT
    assert lib.sphinx_temporal_attention_workspace_size(42, 72, 72, 21, 8) == 2 * 81 * 4
    assert lib.sphinx_sparse_pointwise(p, p, null, null, p, sp.F32, 1, 16, 16, 12, 32, 8, p, p, 4, null, 0,
                                       null) == sp.ERR_UNSUPPORTED


def test_sass_uses_tcgen05_tma_and_mma():
    """The built library is sm_100a code whose conv kernels issue tcgen05 MMAs (UTCHMMA, incl.
    the CTA-pair form), TMA tensor loads (UTMALDG) and bulk copies (UBLKCP), read TMEM with
    LDTM, and whose temporal attention uses warp-level tensor cores (HMMA bf16)."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    so = os.path.join(ROOT, "paper_2511_18672_b200", "libsphinx.so")
    elf = subprocess.run([tool, "-lelf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in elf
    sass = subprocess.run([tool, "-sass", so], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA.2CTA", "UTCHMMA", "UTMALDG.4D", "UTMALDG.3D.2CTA", "UBLKCP", "LDTM",
                     "HMMA.16816.F32.BF16"):
        assert mnemonic in sass, mnemonic
