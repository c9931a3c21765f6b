"""C-ABI boundary checks that run without a GPU: the library loads, exports
every symbol include/monta.h declares, and the Python binding's signature
table covers the header."""
import ctypes as C
import pathlib
import re
import subprocess

from paper_2411_00662_b200 import _lib

HEADER = pathlib.Path(__file__).resolve().parent.parent / "include" / "monta.h"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(moe_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_reports_version():
    lib = _lib.load()
    assert lib.moe_abi_version() == 2  # 2: card view grew (recv_expert_offsets, grad_probs, grad_logits)
    assert lib.moe_dtype_size(_lib.BF16) == 2 and lib.moe_dtype_size(_lib.I64) == 8


def test_every_declared_symbol_is_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (moe_[a-z0-9_]+)", out))
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing


def test_binding_covers_header():
    assert set(header_functions()) <= set(_lib.SIGNATURES), set(header_functions()) - set(_lib.SIGNATURES)


def test_library_has_no_torch_dependency():
    out = subprocess.run(["ldd", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "torch" not in out and "libc10" not in out


def test_sm100a_code_present():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_errors_map_to_exceptions_without_gpu():
    lib = _lib.load()
    out = C.c_double()
    st = lib.moe_lookup_efficiency(None, 1.0, C.byref(out))
    assert st == _lib.ERR_INVALID_ARGUMENT
    assert b"curve" in lib.moe_last_error()


def test_backward_entry_points_validate_without_gpu():
    lib = _lib.load()
    assert lib.moe_route_backward(None, _lib.F32, 4, 2, 3, None, None, None, None) == _lib.ERR_INVALID_ARGUMENT
    assert lib.moe_dispatch_backward(None, _lib.F32, 16, 16, None, 4, 65, None, _lib.F32, 16, None) \
        == _lib.ERR_INVALID_ARGUMENT
    assert b"k <= 64" in lib.moe_last_error()
    assert lib.moe_combine_backward(None, _lib.F32, 16, None, _lib.F32, 16, 16, None, None, _lib.F32, 4, 2,
                                    None, 16, C.c_void_p(1), None) == _lib.ERR_INVALID_ARGUMENT
    assert b"needs the expert rows" in lib.moe_last_error()
    # Nothing to do: no launch, no device needed.
    assert lib.moe_dispatch_backward(None, _lib.F32, 16, 16, None, 0, 2, None, _lib.F32, 16, None) == 0
