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
