"""CPU-side checks of the drop-in boundary: the library builds, loads, exports every symbol the
header declares, and fails loudly (no CPU fallback) when there is no CUDA device."""

import os

import numpy as np
import pytest

import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import _native, lut


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(_native.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build()
    return _native.lib()


def test_header_symbols_all_exported_and_bound(built):
    declared = _native.header_symbols()
    assert len(declared) >= 35
    assert set(declared) == set(_native.SIGNATURES)          # every declared function has a binding
    for name in declared:
        assert hasattr(built, name), name
    assert built.qx_abi_version() == 1


def test_no_cpu_fallback(built):
    try:
        have_gpu = _native.device_count() > 0
    except qx.NativeError:
        have_gpu = False
    if have_gpu:
        pytest.skip("CUDA device present")
    with pytest.raises(qx.NativeError):
        qx.run([qx.Instruction("H", (0,))], 2, "v1")
    with pytest.raises(qx.NativeError):
        qx.canonicalize(qx.SimpleGenerator(1, [1.0], [3]))
    with pytest.raises(qx.NativeError):
        qx.density_expansion(qx.init_z(2))


def test_product_never_imports_the_oracle():
    root = os.path.dirname(_native.HERE)
    for dirpath, _, files in os.walk(_native.HERE):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "stabsim_port" not in text and "qx_oracle" not in text, f
    assert os.path.isdir(os.path.join(root, "oracle"))


def test_host_tables_match_reference(golden):
    # create_lut_1q is bit-identical to the reference's tensor (units.json "lut")
    from paper_2505_03307_b200 import circuit as ir

    for u in golden.load_json("units.json")["lut"]:
        part = ir.divide_instruction(golden.gates(u["gates"]), u["n"])
        mine = lut.create_lut_1q(part)
        assert list(mine.shape) == u["shape"] and part.order == u["order"]
        assert np.array_equal(mine.ravel(), golden.unhex(u["lut"]))
    # CX tables (reference lut.py:108-134) and the known pairs of tests/test_lut.py:126-150
    assert lut.LUT_C.tolist() == [[0, 0, 3, 3], [1, 1, 2, 2], [2, 2, 1, 1], [3, 3, 0, 0]]
    assert lut.LUT_T.tolist() == [[0, 1, 2, 3], [1, 0, 3, 2], [1, 0, 3, 2], [0, 1, 2, 3]]
    assert lut.LUT_SIGN.tolist() == [[1, 1, 1, 1], [1, 1, 1, -1], [1, 1, -1, 1], [1, 1, 1, 1]]
    assert lut.cx_lookup(1, 3) == (2, 2, -1) and lut.cx_lookup(2, 2) == (1, 3, -1)
    for c in range(4):
        for t in range(4):                                    # involution
            c2, t2, s = lut.cx_lookup(c, t)
            c3, t3, s2 = lut.cx_lookup(c2, t2)
            assert (c3, t3) == (c, t) and s * s2 == 1


def test_permutation_classification():
    import math

    assert lut.perm_word(lut.axis_map("H").T) == lut.FIXED_PERMS["H"]
    assert lut.perm_word(lut.gate_branch_block("RZ", math.pi / 4)) is None
    assert lut.perm_word(lut.gate_branch_block("RZ", 0.0)) == lut.IDENTITY_PERM
    # cos(pi/2) = 6e-17 is NOT zero: the reference branches there and so must we
    assert lut.perm_word(lut.gate_branch_block("RX", math.pi / 2)) is None
    # a1/w1/a2/w2 of RZ(theta): X -> cX + sY, Y -> -sX + cY, Z fixed (engine.py:190-202)
    from paper_2505_03307_b200.stabilizer import split_tables

    c, s = math.cos(0.3), math.sin(0.3)
    a1, w1, a2, w2 = split_tables(lut.gate_branch_block("RZ", 0.3))
    assert a1.tolist() == [0, 1, 1, 3] and a2.tolist() == [0, 2, 2, 0]
    assert w1.tolist() == [1.0, c, -s, 1.0] and w2.tolist() == [0.0, s, c, 0.0]
