"""The C-ABI library builds for sm_100a, loads, and exports every declared symbol."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "ekcg_b200.h"


_SASS = {}


def library_sass():
    """cuobjdump -sass of the library, dumped once per test session (the dump takes ~20 s)."""
    from paper_2305_19013_b200 import _lib
    path = _lib.library_path()
    _lib.load()
    if "sass" not in _SASS:
        _SASS["sass"] = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(path)], capture_output=True,
                                       text=True).stdout
    return _SASS["sass"]


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ekcg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared_functions()
    assert "ekcg_spmm_csr" in names and "ekcg_gram" in names and len(names) >= 20


def test_library_exports_every_symbol():
    from paper_2305_19013_b200 import _lib
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(_lib.SIGNATURES)


def test_library_is_sm100a():
    from paper_2305_19013_b200 import _lib
    path = _lib.library_path()
    _lib.load()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(path)], capture_output=True,
                         text=True)
    assert "sm_100a" in out.stdout
    assert "DMMA.8x8x4" in library_sass()  # fp64 tensor-core Gram/update kernels


def test_host_only_queries_without_gpu():
    from paper_2305_19013_b200 import _lib
    assert _lib.query("ekcg_ctrl_bytes") == 80
    assert _lib.query("ekcg_gram_chunks", 262144, 110, 16, 16) >= 1
    assert _lib.query("ekcg_vec_chunks", 1000) == 4
    assert _lib.query("ekcg_launch_count") == 0


def test_invalid_arguments_rejected_without_launch():
    from paper_2305_19013_b200 import _lib
    with pytest.raises(_lib.KernelError, match="invalid argument"):
        _lib.call("ekcg_split", None, None, None, 10, 0, 0, None, None)


def test_cluster_solve_eligibility_and_sass():
    """The one-kernel cluster solve: which (n, t, window) it covers (a host-only query), and that the
    kernel really uses distributed shared memory (st.async completing on a peer's mbarrier) and DMMA."""
    from paper_2305_19013_b200 import _lib
    fits = lambda n, t, w: _lib.query("ekcg_cluster_solve_fits", n, t, w)  # noqa: E731
    assert fits(10000, 8, 2) == 1          # BASELINE config 1 (SRE-CG: window 2)
    assert fits(10000, 8, 4) == 1 and fits(10000, 8, 5) == 0
    assert fits(4096, 16, 2) == 1 and fits(4096, 16, 3) == 0
    assert fits(100, 2, 2) == 1 and fits(100, 1, 1) == 1
    assert fits(10000, 32, 2) == 0         # wide blocks take the launch-per-phase engine
    assert fits(1 << 22, 8, 2) == 0        # beyond n t = 2^22
    sass = library_sass()
    assert "UCGABAR_ARV" in sass and "UCGABAR_WAIT" in sass  # hardware cluster barrier
    assert "STAS.64" in sass                                 # st.async into a peer CTA's shared memory
    assert "SYNCS.ARRIVE.TRANS64" in sass                    # mbarrier expect-tx / complete-tx
