"""CPU-side checks of the boundary: libspc.so builds, loads without a GPU and exports every
entry point include/spc.h declares; host-side argument validation returns the documented
status codes before anything is enqueued."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "spc.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(spc_[a-z0-9_]+)\s*\(", hdr)))


@pytest.fixture(scope="module")
def libspc():
    from paper_2512_00722_b200 import build, spc
    build.build()
    return spc.load_library()


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("spc_score", "spc_topk", "spc_elastic_diff", "spc_gather_kv",
              "spc_sparse_decode_attn"):
        assert s in syms


def test_library_exports_every_declared_symbol(libspc):
    for s in declared_symbols():
        assert hasattr(libspc, s), s
    from paper_2512_00722_b200 import spc
    assert sorted(spc.EXPORTS) == declared_symbols()


def test_status_strings_and_version(libspc):
    assert libspc.spc_version() == 100
    assert libspc.spc_status_string(0) == b"SPC_OK"
    assert b"WORKSPACE" in libspc.spc_status_string(6)


def test_host_validation_without_gpu(libspc):
    """Argument errors are detected on the host, before any CUDA call."""
    P = ctypes.c_void_p(16)
    st = ctypes.c_void_p(0)
    # NULL query
    assert libspc.spc_score(0, None, P, P, 1, 4, 1, 64, 4096, 0.125, 7, P, P, P, P, P, 1 << 20, st) == 1
    # Hq % G != 0
    assert libspc.spc_score(0, P, P, P, 1, 5, 2, 64, 4096, 0.125, 7, P, P, P, P, P, 1 << 20, st) == 2
    # unsupported head dim
    assert libspc.spc_score(0, P, P, P, 1, 4, 1, 96, 4096, 0.125, 7, P, P, P, P, P, 1 << 20, st) == 7
    # workspace too small
    assert libspc.spc_score(0, P, P, P, 1, 4, 1, 64, 4096, 0.125, 7, P, P, P, P, P, 8, st) == 6
    # budget out of range
    assert libspc.spc_topk(P, P, 1, 1, 100, 0, 0, 1, 0, P, None, P, None, P, 1 << 30, st) == 3
    assert libspc.spc_topk(P, P, 1, 1, 100, 5000, 0, 1, 0, P, None, P, None, P, 1 << 30, st) == 3
    assert libspc.spc_elastic_diff(P, P, P, P, 1, 1, 0, None, P, None, P, None, None, st) == 3
    # layer range
    assert libspc.spc_gather_kv(0, P, P, 4, 1, 1, 128, 100, 16, 3, 2, P, P, P, P, P, st) == 4
    ll = ctypes.c_longlong
    assert libspc.spc_gather_kv_strided(0, P, P, ll(1024), ll(0), 4, 1, 1, 128, 16, 3, 2, P, P,
                                        P, P, P, st) == 4
    assert libspc.spc_gather_kv_strided(0, P, P, ll(64), ll(0), 4, 1, 1, 128, 16, 0, 4, P, P,
                                        P, P, P, st) == 2  # row_stride < D
    assert libspc.spc_gather_kv_strided(0, None, P, ll(1024), ll(0), 4, 1, 1, 128, 16, 0, 4, P,
                                        P, P, P, P, st) == 1
    assert libspc.spc_sparse_decode_attn(0, P, P, P, 0, P, P, 2, 0, 3, 1, 4, 1, 128, 100, 16,
                                         0.1, P, None, P, 1 << 30, st) == 4
    assert libspc.spc_score_workspace(1, 32, 32768) > 0
    # one-call step: NULL args / missing workspace are host-side errors
    from paper_2512_00722_b200 import spc
    assert libspc.spc_decode_step(None, st) == 1
    a = spc.StepArgs()
    a.L, a.B, a.Hq, a.G, a.D, a.Smax, a.rows, a.k = 32, 1, 32, 8, 128, 32768, 32768, 2048
    assert libspc.spc_decode_step(ctypes.byref(a), st) == 1  # ws NULL
    a.ws, a.ws_bytes = 16, 8
    assert libspc.spc_decode_step(ctypes.byref(a), st) == 1  # the other buffers NULL: checked first
    for name, _ in spc.StepArgs._fields_:
        if name not in ("L", "B", "Hq", "G", "D", "Smax", "rows", "k", "force_last", "scale",
                        "ws_bytes", "lse", "kv_desc"):
            setattr(a, name, 64)
    assert libspc.spc_decode_step(ctypes.byref(a), st) == 6  # workspace too small
    a.k = 5000
    assert libspc.spc_decode_step(ctypes.byref(a), st) == 3  # budget: before any launch
    assert libspc.spc_decode_step_workspace(32, 1, 32, 8, 128, 32768, 2048) > 0
    # MLA: unsupported latent width, budget, workspace
    assert libspc.spc_mla_sparse_attn(P, P, P, P, P, P, 1, 1, 16, 100, 64, 256, 64, 128, 128, 0.1,
                                      P, None, P, 1 << 30, st) == 7
    assert libspc.spc_mla_sparse_attn(P, P, P, P, P, P, 1, 1, 16, 100, 0, 512, 64, 128, 128, 0.1,
                                      P, None, P, 1 << 30, st) == 3
    assert libspc.spc_mla_workspace(27, 1, 16, 2048) > 0
    # planner: C <= 0 is a capacity error
    c = spc.plan_cfg(10, 100, 2, 1, 1, 1, 2)
    assert libspc.spc_plan_thresholds(ctypes.byref(c), P) == 3


def test_plain_c_program_links_against_the_abi(tmp_path, libspc):
    """The boundary is a C ABI: a C99 program that includes include/spc.h (pedantic, -Werror)
    links against libspc.so and calls it (no GPU needed for these host entry points)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "use_spc.c"
    src.write_text(
        '#include <stdio.h>\n#include "spc.h"\n'
        "int main(void) {\n"
        "  spc_plan_cfg c = {180000000000LL, 16060000000LL, 1.3, 32, 8, 128, 1, 32, 2048, 2};\n"
        "  int64_t th[33];\n"
        "  if (spc_plan_thresholds(&c, th) != SPC_OK) return 2;\n"
        "  printf(\"%d %lld %s\\n\", spc_version(), (long long)th[0], spc_status_string(SPC_E_BUDGET));\n"
        "  return spc_decode_step(NULL, NULL) == SPC_E_NULL ? 0 : 3;\n"
        "}\n")
    exe = tmp_path / "use_spc"
    libdir = os.path.join(root, "paper_2512_00722_b200")
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror",
                           "-I", os.path.join(root, "include"), str(src), "-L", libdir, "-lspc",
                           "-o", str(exe)])
    out = subprocess.check_output([str(exe)], env=dict(os.environ, LD_LIBRARY_PATH=libdir), text=True)
    ver, th0, msg = out.split(maxsplit=2)
    assert int(ver) == 100 and int(th0) == 36788 and "BUDGET" in msg
