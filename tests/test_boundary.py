"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
symbol include/*.h declares, validates shapes with the reference's messages
before touching the GPU, and the C++ mirror header compiles. No GPU compute."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "helix_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hx_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2507_07120_b200 import _lib
    L = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # and the Python binding covers all of them
    assert set(syms) <= set(_lib.EXPORTS), set(syms) - set(_lib.EXPORTS)


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2507_07120_b200", "libhelix_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


def test_sass_uses_bulk_copy_and_hmma():
    so = os.path.join(ROOT, "paper_2507_07120_b200", "libhelix_b200.so")
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass  # cp.async.bulk (TMA bulk engine) in attention and GEMV
    assert "HMMA.16816.F32.BF16" in sass


def test_mla_kernel_uses_tcgen05():
    """The MLA kernel issues paired 5th-gen tensor-core MMAs (UTCHMMA.2CTA),
    moves TMEM with tcgen05.ld/st (LDTM/STTM), commits to mbarriers (UTCBAR)
    and loads latent chunks with 2-SM tensor TMA (UTMALDG.2D.2CTA)."""
    so = os.path.join(ROOT, "paper_2507_07120_b200", "libhelix_b200.so")
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    funcs = sass.split("Function : ")
    mla = [f for f in funcs if f.startswith("_ZN2hx17mla_decode_kernel")]
    assert len(mla) == 2  # bf16 latents (template false) and FP8 latents (true)
    bf16 = [f for f in mla if f.startswith("_ZN2hx17mla_decode_kernelILb0E")]
    fp8 = [f for f in mla if f.startswith("_ZN2hx17mla_decode_kernelILb1E")]
    assert len(bf16) == 1 and len(fp8) == 1
    for op in ("UTCHMMA.2CTA", "LDTM", "STTM", "UTCBAR", "UTMALDG.2D.2CTA", "REDUX.MAX.F32"):
        assert op in bf16[0], op
    # FP8 latents: kind::f8f6f4 paired MMAs (UTCQMMA.2CTA), P packed to e4m3 in registers
    for op in ("UTCQMMA.2CTA", "F2FP.SATFINITE.E4M3.F32.PACK", "LDTM", "UTCBAR", "UTMALDG.2D.2CTA"):
        assert op in fp8[0], op
    assert "UTCHMMA" not in fp8[0]


def test_large_batch_gemv_uses_tcgen05():
    """Batches above 16 run the weight-streaming GEMV on tcgen05 (UTCHMMA with
    TMEM drains, LDTM) fed by TMA bulk copies (UBLKCP); FP8 KV pages widen with
    the e4m3 -> f16 converter (F2FP.F16.E4M3.UNPACK_B), FP4 pages with the
    e2m1 -> f16 converter (F2FP.F16.E2M1.UNPACK_B) and an f16 scale (HMUL2)."""
    so = os.path.join(ROOT, "paper_2507_07120_b200", "libhelix_b200.so")
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    funcs = sass.split("Function : ")
    tc = [f for f in funcs if f.startswith("_ZN2hx14gemv_tc_kernel")]
    assert len(tc) == 4  # N = 32 / 64 batch rows x (2 or 3 activation terms)
    for f in tc:
        for op in ("UTCHMMA", "LDTM", "UBLKCP", "UTCBAR"):
            assert op in f, op
    # FP8 (KV type 1) attention instantiations: 8-row (..Li1ELb0E) and 16-row W16 (..Li1ELb1E) consumers
    att = [f for f in funcs if f.startswith("_ZN2hx18attn_decode_kernel")]
    fp8 = [f for f in att if "ELi1ELb" in f.split("\n", 1)[0]]
    assert any("ELi1ELb1E" in f.split("\n", 1)[0] for f in fp8)
    assert fp8 and all("F2FP.F16.E4M3.UNPACK_B" in f and "HMMA.16816.F32 " in f for f in fp8)
    fp4 = [f for f in att if "ELi2ELb" in f.split("\n", 1)[0]]
    assert any("ELi2ELb1E" in f.split("\n", 1)[0] for f in fp4)
    assert fp4 and all("F2FP.F16.E2M1.UNPACK_B" in f and "HMUL2" in f and "HMMA.16816.F32 " in f for f in fp4)
    # FP8-weight GEMVs (template argument WQ = 1, last) widen e4m3 weights the same
    # way; FP4-weight GEMVs (WQ = 2) widen e2m1 and apply the block scale (HMUL2)
    gemv = [f for f in funcs if f.startswith("_ZN2hx11gemv_kernel")]
    w8 = [f for f in gemv if "Li1EEEv" in f.split("\n", 1)[0]]
    assert w8 and all("F2FP.F16.E4M3.UNPACK_B" in f and "UBLKCP" in f for f in w8)
    w4 = [f for f in gemv if "Li2EEEv" in f.split("\n", 1)[0]]
    assert w4 and all("F2FP.F16.E2M1.UNPACK_B" in f and "HMUL2" in f and "UBLKCP" in f for f in w4)


def test_ctypes_structs_match_c_header(tmp_path):
    """The Python binding's struct layouts equal the C ABI's (sizeof + offsets)."""
    from paper_2507_07120_b200 import _lib
    src = tmp_path / "sz.c"
    src.write_text("""#include <stdio.h>
#include <stddef.h>
#include "helix_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(hx_model_config), sizeof(hx_parallel_config),
         sizeof(hx_runtime_config), sizeof(hx_engine_info), offsetof(hx_model_config, kv_latent),
         offsetof(hx_parallel_config, ep));
  return 0;
}
""")
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)], text=True).split()]
    import ctypes as C
    want = [C.sizeof(_lib.ModelConfig), C.sizeof(_lib.ParallelConfig), C.sizeof(_lib.RuntimeConfig),
            C.sizeof(_lib.EngineInfo), _lib.ModelConfig.kv_latent.offset, _lib.ParallelConfig.ep.offset]
    assert got == want


@pytest.mark.parametrize("dims,tpa,kvp,msg", [
    ((4, 3, 8), 1, 1, "multiple of kv_heads"),
    ((4, 2, 8), 4, 1, "tpa must divide kv_heads"),
    ((4, 2, 8), 2, 3, "divide the hidden width"),
    ((4, 2, 8), 0, 1, "tpa and kvp must be >= 1"),
    ((4, 2, 8), 1, 0, "cache dimensions must be >= 1"),
    ((32, 2, 8), 1, 128, "kvp > 64 is not supported"),
])
def test_reference_validation_without_gpu(dims, tpa, kvp, msg):
    """Same checks, order and messages as attention.hpp:239-240, 431-437 --
    raised before any CUDA call, so they hold on a CPU-only host."""
    import paper_2507_07120_b200 as P
    with pytest.raises(ValueError, match=msg):
        P.DecodeHarness(dims, tpa, kvp, 16, 1)


def test_no_cpu_fallback():
    """Without a usable GPU the product fails loudly instead of computing on the CPU."""
    import paper_2507_07120_b200 as P
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(P.CudaError):
        P.DecodeHarness((4, 2, 8), 2, 4, 16, 42)


def test_cpp_mirror_header_compiles():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")])


def test_round_robin_closed_form_matches_oracle():
    """kv_layout.cuh rr_rank/rr_row/rr_count == the reference cursor walk."""
    from tests import oracle_py as O
    for kvp, chunk in [(1, 16), (4, 16), (3, 7), (8, 1), (2, 5)]:
        h = O.Harness(4 * 6, 2, 8, 1, kvp, chunk, 1)  # hidden 192: divisible by kvp in {1,2,3,4,8}
        n = 137
        h.grow_random(n, O.Rng(9))
        ranks, rows = h.token_order()
        g = np.arange(n)
        np.testing.assert_array_equal(ranks, (g // chunk) % kvp)
        np.testing.assert_array_equal(rows, (g // (chunk * kvp)) * chunk + g % chunk)
        for r in range(kvp):
            full, rem = divmod(n, chunk * kvp)
            assert h.effective_tokens(r) == full * chunk + min(max(rem - r * chunk, 0), chunk)
