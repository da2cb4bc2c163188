"""Host-side checks of the C-ABI library (no GPU needed): libzinc.so loads, exports
every symbol include/zinc.h declares, and validates arguments before touching
the device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "zinc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:zinc|ckks)_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    import paper_2408_07304_b200 as Z
    assert sorted(Z.EXPORTED_SYMBOLS) == declared_symbols()


def test_library_loads_and_exports_every_symbol():
    import paper_2408_07304_b200 as Z
    lib = Z.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_argument_validation_without_gpu():
    import paper_2408_07304_b200 as Z
    lib = Z.lib()
    h = ctypes.c_void_p()
    bits = (ctypes.c_int * 3)(36, 36, 36)
    assert lib.zinc_ctx_create(11, 3, bits, 30, 0, ctypes.byref(h)) == -1      # log_n < 12
    assert b"log_n" in lib.zinc_last_error()
    assert lib.zinc_ctx_create(12, 0, bits, 30, 0, ctypes.byref(h)) == -1      # L = 0
    bad = (ctypes.c_int * 3)(36, 61, 36)
    assert lib.zinc_ctx_create(12, 3, bad, 30, 0, ctypes.byref(h)) == -1       # 61-bit limb
    assert lib.zinc_ctx_create(12, 3, None, 30, 0, ctypes.byref(h)) == -1      # null
    # null context on every call
    assert lib.zinc_keygen(None, 1, None, None, None, None) == -1
    assert lib.zinc_encrypt_batch(None, None, 0, 0, None, 1, 0, 0, None, None) == -1
    assert lib.ckks_decrypt_batch(None, None, 0, None, 1, None, None, None, None) == -1
    # scheme validation happens before any device work
    assert lib.zinc_ctx_create_scheme(12, 3, bits, 3, 65537, 0, 0, ctypes.byref(h)) == -1    # bad scheme
    assert b"scheme" in lib.zinc_last_error()
    assert lib.zinc_ctx_create_scheme(12, 3, bits, 1, 1, 0, 0, ctypes.byref(h)) == -1        # t < 2
    assert lib.zinc_ctx_create_scheme(12, 3, bits, 2, 1 << 32, 0, 0, ctypes.byref(h)) == -1  # t >= 2^32
    assert b"plain modulus" in lib.zinc_last_error()
    lib.zinc_launch_count_reset()
    assert lib.zinc_launch_count() == 0


def test_product_path_does_not_import_oracle():
    """The product package and its C sources never reference oracle/."""
    pkg = os.path.join(ROOT, "paper_2408_07304_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "oracle.h" not in text and "liboracle" not in text, f
