"""CPU-side checks of the C ABI (no GPU needed): the library loads, exports every
symbol include/magicpig.h declares, and its host-side size / validation logic
is consistent with the layout documented in the header."""
from __future__ import annotations

import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "magicpig.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(magicpig_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2410_16179_b200 import binding
    return binding.lib()


def test_header_symbols_exported(lib):
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in magicpig.h but not exported"


def test_binding_covers_header():
    from paper_2410_16179_b200 import binding
    assert set(_declared()) == set(binding.exported_symbols())


def test_version_and_strerror(lib):
    from paper_2410_16179_b200 import binding
    assert "sm_100a" in binding.version()
    for code in range(0, -8, -1):
        assert lib.magicpig_strerror(code)


def test_config_validation():
    from paper_2410_16179_b200 import binding
    ok = binding.make_config()
    assert binding.lib().magicpig_validate_config(C.byref(ok)) == 0
    bad = [dict(K=0), dict(K=17), dict(L=1), dict(min_collisions=3), dict(mips=2)]
    for kw in bad:
        c = binding.make_config(**kw)
        assert binding.lib().magicpig_validate_config(C.byref(c)) != 0, kw
    c = binding.make_config()
    c.head_dim = 64
    assert binding.lib().magicpig_validate_config(C.byref(c)) != 0


@pytest.mark.parametrize("K,L", [(10, 150), (8, 75), (11, 300), (7, 35), (16, 9), (1, 2), (3, 5)])
def test_codes_words_layout(K, L):
    """codes_words = units * ceil(n/1024) * KLq * 128 with KLq = ceil(L/TG)*QG,
    TG = 4/gcd(K,4) tables, QG = K/gcd(K,4) quads per group (header layout)."""
    from math import gcd
    from paper_2410_16179_b200 import binding
    cfg = binding.make_config(K=K, L=L)
    for B, Hkv, n in [(1, 1, 1), (1, 8, 16384), (2, 3, 1025), (1, 1, 0)]:
        TG, QG = 4 // gcd(K, 4), K // gcd(K, 4)
        KLq = -(-L // TG) * QG
        want = B * Hkv * (-(-n // 1024)) * KLq * 128
        assert binding.codes_words(cfg, B, Hkv, n) == want
        # bytes ~= n * K * L / 8 per unit (plus padding)
        if n >= 1024:
            assert want * 4 >= B * Hkv * n * K * L / 8


@pytest.mark.parametrize("K,L", [(10, 150), (7, 35), (14, 6), (3, 5)])
def test_bucket_tables_words_layout(K, L):
    """bucket_tables_words = units * (L*(2^K+1) int32 offsets + ids): the L*n ids take 16 bits each when
    n <= 65536 (the paper's int16 table entries; ceil(L*n/2) words), 32 bits above (header layout)."""
    from paper_2410_16179_b200 import binding
    cfg = binding.make_config(K=K, L=L)
    for B, Hkv, n in [(1, 1, 1), (1, 8, 16384), (2, 3, 1025), (1, 1, 65536), (1, 2, 65537), (1, 1, 100001)]:
        ids = -(-(L * n) // 2) if n <= 65536 else L * n
        assert binding.bucket_tables_words(cfg, B, Hkv, n) == B * Hkv * (L * ((1 << K) + 1) + ids)
    assert binding.bucket_tables_words(binding.make_config(K=15, L=L), 1, 1, 1000) == 0  # K <= 14 only


def test_workspace_sizes_positive():
    from paper_2410_16179_b200 import binding
    cfg = binding.make_config()
    assert binding.build_workspace_bytes(cfg, 1, 8, 16384) > 8 * 16384 * 144 * 2
    assert binding.decode_workspace_bytes(cfg, 1, 32, 8, 16384) > 0
    assert binding.decode_workspace_bytes(cfg, 1, 30, 8, 16384) == 0  # Hq not a multiple of Hkv
