"""The C-ABI library loads and exports every symbol include/tga.h declares
(no compute calls -- CPU only)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "tga.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tga_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for f in ["tga_instance_create", "tga_solution_load", "tga_eval", "tga_best_move", "tga_apply_move"]:
        assert f in names


def test_library_exports_every_declared_symbol():
    from paper_2506_17357_b200 import build
    build.build()
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2506_17357_b200", "libtga.so"))
    for name in _declared():
        assert hasattr(lib, name), name


def test_binding_symbol_table_matches_header():
    from paper_2506_17357_b200 import tga
    assert sorted(tga._SYMBOLS) == _declared()


def test_variant_tables_agree_with_oracle():
    """Variant ids are the tie-break rank on both sides (kept in sync by this
    test, not by shared code)."""
    import oracle as O
    from paper_2506_17357_b200 import tga
    assert tga.N_VARIANTS == O.N_VARIANTS
    assert tga.V_RELOCATE == O.V_RELOC and tga.V_SWAP == O.V_SWAP
    assert tga.V_IRELOCATE == O.V_IRELOC and tga.V_ISWAP == O.V_ISWAP
    assert tga.V_OROPT_REV == O.V_RELOC_REV and tga.V_CROSS_REV == O.V_CROSS_REV
    hdr = open(os.path.join(ROOT, "include", "tga.h")).read()
    ids = {name: int(val) for name, val in re.findall(r"TGA_V_([A-Z0-9_]+)\s*=\s*(\d+)", hdr)}
    assert ids["OROPT2R"] == O.V_RELOC_REV[2] and ids["CROSS33R"] == O.V_CROSS_REV[3]
    assert ids["ISWAP33"] == O.V_ISWAP[(3, 3)] and ids["CROSS33"] == O.V_SWAP[(3, 3)]
    assert f"TGA_N_VARIANTS = {O.N_VARIANTS}" in hdr
    assert len(tga.VARIANT_NAMES) == O.N_VARIANTS


def test_version_and_error_strings_without_gpu():
    from paper_2506_17357_b200 import tga
    assert "sm_100a" in tga.version()
    assert isinstance(tga.lib().tga_last_error(), bytes)


def test_instance_argument_validation_without_gpu():
    """Argument checks happen before any device call."""
    from paper_2506_17357_b200 import tga
    d = np.array([[0, 1], [2, 0]], dtype=np.int32)
    with pytest.raises(tga.TgaError) as e:
        tga.Instance(d, [0, 1], 10)
    assert e.value.code == -4  # asymmetric -> unsupported
    d = np.array([[0, 1], [1, 0]], dtype=np.int32)
    with pytest.raises(tga.TgaError) as e:
        tga.Instance(d, [0, -1], 10)
    assert e.value.code == -1


def test_key_decode_roundtrip():
    from paper_2506_17357_b200 import tga
    for s in [-5, 0, 7, -2 ** 31, 2 ** 31 - 1]:
        ordv = (s & 0xFFFFFFFF) ^ 0x80000000
        assert tga.decode_key((ordv << 32) | 123) == (s, 123)


def test_fast_tile_order_is_a_bijection_onto_the_plan():
    """The tile kernel decodes its tile order arithmetically (no plan table): for
    U = 8 and 16 and many slot counts, t -> (I, J) enumerates exactly the tiles of
    the upper triangle, I U < Qp, J 128 < Qp, I U < 128 J + 127, each once
    (host logic of libtga.so; no GPU needed)."""
    import ctypes as C
    from paper_2506_17357_b200 import tga as T
    L = T.lib()
    f = L.tga_debug_fast_tile
    f.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    I, J = C.c_int32(), C.c_int32()
    for U in (8, 16):
        R = 128 // U
        for Qp in list(range(1, 400, 7)) + [1176, 2352, 10870, 40000]:
            nI, nJ = -(-Qp // U), -(-Qp // 128)
            plan = {(i, j) for i in range(nI) for j in range(nJ) if i * U < 128 * j + 127}
            n = nI + R * nJ * (nJ - 1) // 2
            assert n == len(plan), (U, Qp)
            got = set()
            for t in range(n):
                assert f(t, nI, R, C.byref(I), C.byref(J)) == 0
                got.add((I.value, J.value))
            assert got == plan, (U, Qp)


def test_ns_tile_order_is_a_bijection_onto_the_plan():
    """The north-star sweep kernel's tile order (tga_ns.cu, decoded arithmetically;
    tiles of TU = 16 / 32 / 64 rows x 128 columns, RB = 128 / TU row bands per column
    band): t -> (I, J) enumerates every tile that holds a cell of the upper triangle,
    each once; the lightest diagonal tiles last (host logic; no GPU)."""
    import ctypes as C
    from paper_2506_17357_b200 import tga as T
    L = T.lib()
    f = L.tga_debug_ns_tile
    f.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    I, J = C.c_int32(), C.c_int32()
    for TU in (16, 32, 64):
        RB = 128 // TU
        for Qp in list(range(1, 600, 11)) + [1176, 2352, 2944, 10870, 40000]:
            nI, nJ = -(-Qp // TU), -(-Qp // 128)
            plan = {(i, j) for i in range(nI) for j in range(nJ) if i * TU < 128 * j + 127}
            n = nI + RB * nJ * (nJ - 1) // 2
            assert n == len(plan), (TU, Qp)
            got = []
            for t in range(n):
                assert f(t, nI, nJ, RB, C.byref(I), C.byref(J)) == 0
                got.append((I.value, J.value))
            assert set(got) == plan and len(set(got)) == n, (TU, Qp)
            n3 = nI // RB
            # diagonal tiles that do not close their band lead, the lightest close the plan
            assert all(j == i // RB and i % RB != RB - 1 for i, j in got[:nI - n3]), (TU, Qp)
            assert all(j == i // RB and i % RB == RB - 1 for i, j in got[n - n3:]), (TU, Qp)
