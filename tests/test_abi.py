"""C-ABI library: builds, loads, exports every symbol include/moe.h declares,
and the host-only entry points (config validation, size queries) behave.
No compute calls here (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "moe.h")
LIB = os.path.join(ROOT, "paper_2211_15841_b200", "libmoe.so")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(moe_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "run make"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (moe_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert len(declared_symbols()) >= 20


def test_binding_signatures_cover_header():
    from paper_2211_15841_b200._lib import SIGNATURES
    assert sorted(SIGNATURES) == declared_symbols()


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sass_has_tcgen05_and_tma():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out       # tcgen05.mma
    assert "UTMALDG" in out       # TMA loads
    assert "LDTM" in out          # tcgen05.ld
    assert "HMMA" not in re.sub(r"UTCHMMA", "", out)  # no legacy mma.sync path


def _cfg(**kw):
    from paper_2211_15841_b200.api import make_config
    base = dict(tokens=1024, hidden=256, num_experts=4, top_k=1, ffn_hidden=512)
    base.update(kw)
    return make_config(**base)


def test_check_config_and_errors():
    from paper_2211_15841_b200 import api
    from paper_2211_15841_b200._lib import lib
    assert api.moe_check_config(_cfg()) == 0
    assert api.moe_check_config(_cfg(top_k=5)) == 1               # k > E
    assert b"top_k" in lib.moe_last_error()
    assert api.moe_check_config(_cfg(ffn_hidden=500)) == 2        # f % bs
    assert api.moe_check_config(_cfg(block_size=64, ffn_hidden=512)) == 3   # GPU path is bs=128
    assert api.moe_check_config(_cfg(hidden=200)) == 3
    assert api.moe_check_config(_cfg(act=7)) == 1
    assert lib.moe_check_config(None) == 1


def test_size_queries_match_oracle_bound():
    from oracle import moe_oracle as O
    from paper_2211_15841_b200 import api
    for T, k, E in [(1024, 1, 4), (32768, 1, 64), (8192, 2, 64), (3, 1, 64), (1, 1, 1)]:
        cfg = _cfg(tokens=T, top_k=k, num_experts=E, hidden=512, ffn_hidden=2048)
        rows = api.moe_max_padded_rows(cfg)
        assert rows == O.max_padded_rows(T, k, E, 128)
        assert api.moe_max_nnz_blocks(cfg) == rows // 128 * 16
        assert api.moe_workspace_bytes(cfg) > 0


def test_null_arguments_rejected_without_launch():
    from paper_2211_15841_b200._lib import lib
    cfg = _cfg()
    st = lib.moe_gather(ctypes.byref(cfg), None, None, None, None)
    assert st == 1 and b"NULL" in lib.moe_last_error()


def test_check_config_formulation_fields():
    """capacity / renormalize / aux_loss_coeff (NEXT-4) are validated on the host;
    moe_expert_capacity matches the oracle's ceil(T*cf/E)."""
    import math
    from oracle import moe_oracle as O
    from paper_2211_15841_b200 import api
    from paper_2211_15841_b200._lib import lib
    assert api.moe_check_config(_cfg(capacity=3, renormalize=True, aux_loss_coeff=0.01)) == 0
    assert api.moe_check_config(_cfg(capacity=-1)) == 1 and b"capacity" in lib.moe_last_error()
    cfg = _cfg()
    cfg.renormalize = 2
    assert api.moe_check_config(cfg) == 1 and b"renormalize" in lib.moe_last_error()
    for bad in (-0.5, math.nan, math.inf):
        assert api.moe_check_config(_cfg(aux_loss_coeff=bad)) == 1
    for T, E, cf in [(8, 4, 1.0), (1000, 64, 1.5), (32768, 64, 2.0), (7, 3, 0.5), (10, 4, 0.0)]:
        want = O.expert_capacity(T, E, cf) if cf > 0 else 0
        assert api.moe_expert_capacity(T, E, cf) == want
    # workspace offset 5 (aux region) exists and leaves room for {loss, E coefficients}
    cfg = _cfg(num_experts=64, hidden=512, ffn_hidden=2048)
    off = lib.moe_workspace_offset(ctypes.byref(cfg), 5)
    assert 0 < off and off + 4 * 65 <= api.moe_workspace_bytes(cfg)


def _gelu_argmin(O):
    """argmin of the oracle's gelu: the root of its act_grad on [-1.5, -0.3] (bisection)."""
    lo, hi = -1.5, -0.3
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        lo, hi = (mid, hi) if O.act_grad(O.ACT_GELU, mid) < 0 else (lo, mid)
    return 0.5 * (lo + hi)


def _encode_r24(O, h):
    """The branch code of moe.h / DESIGN R24, written from its description: A = gelu(h)
    in fp32; h >= 0: RNE bf16; h < 0: sign set, the bf16 of A's magnitude whose
    mantissa LSB = (h < argmin gelu) nearest to A."""
    import numpy as np
    a = O.act(O.ACT_GELU, h).astype(np.float32)
    bits = a.view(np.uint32)
    rne = ((bits + 0x7FFF + ((bits >> 16) & 1)) >> 16).astype(np.uint32)
    trunc = (bits >> 16) | 0x8000
    b = (h < _gelu_argmin(O)).astype(np.uint32)
    neg = np.where((trunc & 1) == b, trunc, trunc + 1)
    return np.where(h < 0, neg, rne).astype(np.uint16)


def test_act_code_decode_matches_oracle_derivative():
    """R24: act'(H) as the SDD^T decodes it from the branch-coded A (the
    library's table, host copy) against the oracle's float64 act'(h), for h
    over several scales; special cases exact; relu = (A > 0)."""
    import numpy as np
    from oracle import moe_oracle as O
    from paper_2211_15841_b200 import api
    rng = np.random.default_rng(7)
    for sigma in (0.25, 1.0, 3.0):
        h = rng.standard_normal(200_000) * sigma
        got = api.moe_act_code_decode_host(api.ACT_GELU, _encode_r24(O, h)).astype(np.float64)
        want = O.act_grad(O.ACT_GELU, h)
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert rel < 6e-3, (sigma, rel)          # bf16-storage level (act' itself in bf16: ~2e-3)
        assert np.abs(got - want).max() < 0.03   # worst case: near gelu's minimum (act' ~ sqrt(A - A_min))
    # exact special cases: act'(0) = 1/2, act' = 1 for large h, ~0 far left of the minimum
    h = np.array([0.0, 8.0, 20.0, 1e4, -12.0, -40.0])
    got = api.moe_act_code_decode_host(api.ACT_GELU, _encode_r24(O, h))
    np.testing.assert_allclose(got[:4], [0.5, 1.0, 1.0, 1.0], atol=1e-3)
    assert np.abs(got[4:]).max() < 2e-3
    # each branch of a negative A decodes to its own side of the minimum
    xm = _gelu_argmin(O)
    h = np.array([xm + 0.3, xm - 0.3, xm + 0.05, xm - 0.05])
    got = api.moe_act_code_decode_host(api.ACT_GELU, _encode_r24(O, h))
    assert got[0] > 0.05 and got[1] < -0.05 and got[2] > 0 and got[3] < 0
    # relu: act' = A > 0 on plain RNE bf16 of relu(h)
    h = rng.standard_normal(1000)
    a = np.maximum(h, 0).astype(np.float32).view(np.uint32)
    got = api.moe_act_code_decode_host(api.ACT_RELU, ((a + 0x7FFF + ((a >> 16) & 1)) >> 16).astype(np.uint16))
    np.testing.assert_array_equal(got, (h > 0).astype(np.float32))
