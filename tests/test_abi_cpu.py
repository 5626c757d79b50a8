"""CPU-side checks of the product boundary: the C-ABI library loads and exports every
symbol include/mpfem_b200.h declares; host-side generators equal the reference-semantics
oracle bitwise; config validation raises ConfigError before any device work; without a
GPU every compute entry fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2410_12614_b200 as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "mpfem_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mpfem_b200_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(mp.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert b"sm_100a" in mp.lib().mpfem_b200_version()


def test_sm100a_code_in_library():
    data = open(mp.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


@pytest.mark.parametrize("kind,seed", [(0, 1), (0, 42), (1, 3)])
def test_generators_match_oracle(oracle, kind, seed):
    a = mp.gen_tets(kind, seed, 3000)
    b = oracle.gen_tets(kind, seed, 3000)
    assert np.array_equal(a[0], b[0])
    if kind == 1:
        assert np.array_equal(a[1], b[1])


def test_structured_mesh_matches_oracle(oracle):
    for dims, jit, seed in (((5, 4, 3), 0.15, 9), ((2, 2, 2), 0.0, 1), ((1, 1, 7), 0.3, 4)):
        a = mp.structured_tet_mesh(*dims, 1.0, jit, seed)
        b = oracle.structured_tet_mesh(*dims, 1.0, jit, seed)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    with pytest.raises(mp.ConfigError):
        mp.structured_tet_mesh(0, 1, 1)
    with pytest.raises(mp.ConfigError):
        mp.structured_tet_mesh(1, 1, 1, 1.0, 0.5)


def test_config_validation_before_device():
    # kernels.cpp:29-40: matrix engine needs u_s = bf16 and u_q = fp32; batch >= 1
    with pytest.raises(mp.ConfigError):
        mp.make_setup(2, mp.KernelConfig(u_s=mp.Fmt.fp16, u_q=mp.Fmt.fp32, engine=mp.EngineKind.matrix))
    with pytest.raises(mp.ConfigError):
        mp.make_setup(2, mp.KernelConfig(n_batch=0))
    with pytest.raises(mp.ConfigError):
        mp.make_setup(0, mp.KernelConfig())
    with pytest.raises(mp.ConfigError):  # action_kernel needs an action-mode config
        mp.action_kernel(type("S", (), {"config": mp.KernelConfig()})(), None, None)
    with pytest.raises(mp.ConfigError):  # bf16 accumulation has no B200 path
        mp.make_setup(2, mp.KernelConfig(u_q=mp.Fmt.bf16, u_s=mp.Fmt.bf16))


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(mp.RuntimeFailure):
        mp.make_setup(2, mp.mode_config("mixed", mp.FormKind.poisson))


def test_mode_table():
    c = mp.mode_config("mixed_bf16", mp.FormKind.mass)
    assert (c.u_p, c.u_g, c.u_q, c.u_s, c.engine) == (mp.Fmt.fp32, mp.Fmt.fp32, mp.Fmt.fp32,
                                                      mp.Fmt.bf16, mp.EngineKind.matrix)
    c = mp.mode_config("mixed", mp.FormKind.poisson, geometry_fp64=True)
    assert c.u_g == mp.Fmt.fp64 and c.u_s == mp.Fmt.fp16
