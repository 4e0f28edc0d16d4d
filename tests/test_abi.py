"""CPU checks of the C-ABI boundary: the library builds, loads without a GPU, and
exports every function include/ckks.h declares; the binding mirrors the same names."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ckks.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ckks_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_north_star_calls():
    fns = header_functions()
    for name in ("ckks_ctx_create", "ckks_encode", "ckks_encrypt", "ckks_decrypt", "ckks_add", "ckks_mul_plain",
                 "ckks_mul_relin", "ckks_rescale", "ckks_rotate", "ckks_privft_infer", "ckks_total_sum",
                 "ckks_ntt", "ckks_modadd_gathered"):
        assert name in fns


def test_library_exports_every_declared_symbol():
    from paper_1908_06972_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)  # no CUDA call happens at load time
    missing = [f for f in header_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_binding_mirrors_header():
    from paper_1908_06972_b200 import ckks
    assert sorted(ckks.EXPORTS) == header_functions()
    ckks.lib()  # loads and sets argtypes for every export


def test_library_is_sm100a_only():
    """The fat binary carries sm_100a SASS (no PTX/JIT fallback for other archs)."""
    import subprocess
    from paper_1908_06972_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.build()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in ln for ln in out.splitlines() if ln.strip())
