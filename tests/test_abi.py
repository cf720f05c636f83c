"""CPU tests of the C-ABI boundary: the engine library loads without a GPU
and exports every entry point the public headers declare; structs keep the
layout the Python mirror assumes; the host-side generator matches the
reference generator bit for bit."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2503_07680_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("hbp_b200.h", "hbp_b200_testing.h")]


def declared_functions():
    names = set()
    for h in HEADERS:
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(hbp_[a-z0-9_]+)\s*\(", text):
            names.add(m.group(1))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    lib = abi.load_library()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert len(declared_functions()) >= 30


def test_no_gpu_context_fails_loudly():
    # on a CPU-only box creating a context reports a CUDA error, never a fallback
    lib = abi.load_library()
    h = C.c_void_p()
    rc = lib.hbp_ctx_create(0, C.byref(h))
    import torch
    if torch.cuda.is_available():
        assert rc == abi.HBP_OK
        lib.hbp_ctx_destroy(h)
    else:
        assert rc == abi.HBP_ERR_CUDA


def test_struct_sizes():
    # offsets of the C structs as compiled (x86-64 SysV)
    assert C.sizeof(abi.GroupConfig) == 16
    assert C.sizeof(abi.HardwareProfile) == 88
    assert C.sizeof(abi.PlanOptions) == 40  # strategy 16 + 3 x int32 + pad + uint64
    assert C.sizeof(abi.Samples) == 40


def test_defaults_match_reference_header():
    lib = abi.load_library()
    p = abi.HardwareProfile()
    lib.hbp_hardware_profile_defaults(C.byref(p))
    q = abi.default_profile()
    for f, _ in abi.HardwareProfile._fields_:
        assert getattr(p, f) == getattr(q, f), f


@pytest.mark.parametrize("n,short,lf,long_,seed", [
    (200_000, "lognormal:7.2:0.7", 0.02, "uniform:16385:131072", 20250515),
    (50_000, "lognormal:8.5:1.4", 0.0, "", 42),
    (1001, "normal:100:30", 0.3, "constant:5", 3),
])
def test_synth_matches_reference_generator(oracle, n, short, lf, long_, seed):
    lib = abi.load_library()
    out = np.zeros(n, dtype=np.int64)
    err = C.create_string_buffer(256)
    rc = lib.hbp_synth_lengths(C.c_int64(n), short.encode(), C.c_double(lf), long_.encode(), C.c_int64(131072),
                               C.c_uint64(seed), out.ctypes.data_as(C.POINTER(C.c_int64)), err, 256)
    assert rc == 0
    assert np.array_equal(out, oracle.synth(n, short, lf, long_, 131072, seed))


def test_synth_errors():
    lib = abi.load_library()
    out = np.zeros(4, dtype=np.int64)
    err = C.create_string_buffer(256)
    rc = lib.hbp_synth_lengths(C.c_int64(4), b"gamma:1:2", C.c_double(0), b"", C.c_int64(10), C.c_uint64(0),
                               out.ctypes.data_as(C.POINTER(C.c_int64)), err, 256)
    assert rc == abi.HBP_ERR_VALIDATION and err.value == b"unknown distribution family: gamma"


def _c3_like_candidates():
    """C3's candidate order (sweep.make_candidates) with ckpt 0: the dealing
    only reads the length sets."""
    import itertools
    out = []
    smaller = [512, 1024, 2048, 4096, 8192, 16384, 32768, 65536]
    for r in range(len(smaller) + 1):
        for subset in itertools.combinations(smaller, r):
            ls = list(subset) + [131072]
            for sp in (1, 2, 4, 8):
                for _gc in (True, False):
                    out.append(([(l, 1 if i == 0 else sp, 0) for i, l in enumerate(ls)], ls[0]))
    return out


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_sweep_shard_matches_python_dealing(world):
    # hbp_sweep_sharded deals length sets in C++; sweep.shard() is the same
    # rule on the Python (gloo) path: both must give every rank the same share
    from paper_2503_07680_b200 import sweep
    lib = abi.load_library()
    cands = _c3_like_candidates()
    garr, offs, _ = abi.flatten_candidates(cands)
    lib.hbp_test_sweep_shard.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p,
                                         C.POINTER(C.c_int64)]
    seen = []
    for rank in range(world):
        out = np.zeros(len(cands), dtype=np.int64)
        n = C.c_int64()
        assert lib.hbp_test_sweep_shard(garr, offs.ctypes.data, len(cands), rank, world, out.ctypes.data,
                                        C.byref(n)) == abi.HBP_OK
        got = out[:n.value].tolist()
        assert got == sweep.shard(cands, rank, world)
        seen += got
    assert sorted(seen) == list(range(len(cands)))
