"""The C-ABI library: it builds for sm_100a, loads, exports every symbol the
header declares, and reports errors the way the reference does (ValueError
for arguments, RuntimeError for device state).  No compute calls here."""

import ctypes as C
import os
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "hogbatch_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\*?\s*(hb_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2004_08771_b200 import _native, build

    if not _native.LIB_PATH.exists():
        build.build()
    return _native.load()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("hb_ctx_create", "hb_set_weights_f64", "hb_train_step", "hb_merge_grad_into_f64",
                 "hb_eval_loss_sum", "hb_stage_csr", "hb_merge_allreduce", "hb_last_error"):
        assert must in syms
    assert len(syms) >= 25


def test_every_declared_symbol_is_exported_and_typed(lib):
    from paper_2004_08771_b200 import _native

    nm = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(hb_\w+)", nm))
    for s in declared_symbols():
        assert s in exported, s
        assert s in _native.SIGNATURES, f"{s} missing from the ctypes binding"
        assert hasattr(lib, s)


def test_library_is_sm100a_native(lib):
    from paper_2004_08771_b200 import _native

    out = subprocess.run(["cuobjdump", "-sass", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", str(_native.LIB_PATH)], capture_output=True,
                                       text=True).stdout
    assert "UTCHMMA" in out  # tcgen05.mma
    assert "UTMALDG" in out  # TMA loads
    assert "LDTM" in out  # tcgen05.ld (TMEM -> registers)
    assert "HMMA" not in re.sub(r"UTCHMMA", "", out)  # no legacy mma.sync path


def test_version_and_errors(lib):
    import paper_2004_08771_b200 as hb

    assert b"sm_100a" in lib.hb_version()
    n = hb.device_count()
    assert n >= 0
    # argument errors are ValueError and are checked before touching a device
    with pytest.raises(ValueError, match="layer sizes"):
        hb.GpuReplica((5, 0, 2), 8)
    with pytest.raises(ValueError, match="classes"):
        hb.GpuReplica((5, 4, 1), 8)
    with pytest.raises(ValueError):
        hb.GpuReplica((5, 4, 2), 0)
    with pytest.raises(ValueError, match="sparse"):
        hb.GpuReplica((5, 2), 8, sparse=True)
    h = C.c_void_p()
    assert lib.hb_ctx_create(C.byref(h), 0, 2, None, 8, 0) == 1
    assert b"null" in lib.hb_last_error()
    if n == 0:
        with pytest.raises(RuntimeError, match="no CUDA device"):
            hb.GpuReplica((5, 4, 2), 8)


def test_product_path_has_no_oracle_or_fallback():
    """The shipped package never imports the test oracle or a CPU math path."""
    pkg = ROOT / "paper_2004_08771_b200"
    for f in pkg.glob("*.py"):
        src = f.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), f
        assert "import hogtrain" not in src or f.name == "workers.py", f  # install() only rebinds
    missing = ROOT / "nonexistent.so"
    code = (f"import os; os.environ['HOGBATCH_B200_LIB']={str(missing)!r}\n"
            "from paper_2004_08771_b200 import _native\n"
            "try:\n    _native.load()\nexcept _native.NativeLibraryMissing as e:\n    print('LOUD', e)\n")
    out = subprocess.run(["python", "-c", code], capture_output=True, text=True, cwd=ROOT).stdout
    assert out.startswith("LOUD")


def test_host_merge_pool_resizes(lib):
    """hb_host_merge_threads (host only, no GPU): resize and restore the merge pool."""
    assert lib.hb_host_merge_threads(3, 0) == 0
    assert lib.hb_host_merge_threads(1, 100) == 0
    assert lib.hb_host_merge_threads(0, 0) != 0  # invalid
    assert lib.hb_host_merge_threads(4, 20000) == 0


def test_host_merge_pool_runs_every_part_once(lib):
    """The merge pool's tickets carry their job: across 20000 back-to-back jobs
    of growing and shrinking part counts, with the pool spinning (stale
    workers race the next job) and sleeping, every part runs exactly once."""
    for threads, spin in ((8, 20000), (3, 0), (12, 200)):
        assert lib.hb_host_merge_threads(threads, spin) == 0
        err = C.c_int64(-1)
        assert lib.hb_host_pool_selftest(20000, C.byref(err)) == 0
        assert err.value == 0, (threads, spin, err.value)
    assert lib.hb_host_merge_threads(max(2, min(12, (os.cpu_count() or 4) * 3 // 4)), 20000) == 0
