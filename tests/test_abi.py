"""C-ABI checks that need no GPU: the library builds for sm_100a, loads,
exports every symbol include/hjcd.h declares, and validates arguments on the
host before touching CUDA."""
import ctypes as C
import os
import re
import subprocess

import pytest

from params import DEFAULTS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "hjcd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hjcd_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(hjcd_lib):
    decl = header_symbols()
    assert len(decl) >= 15
    L = hjcd_lib.lib()
    missing = [s for s in decl if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(hjcd_lib.EXPORTS) == decl


def test_library_is_sm100a(hjcd_lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", hjcd_lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert hjcd_lib.version().startswith("hjcd")


def test_config_default_matches_design(hjcd_lib):
    c = hjcd_lib.default_config()
    for k, v in DEFAULTS.items():
        name = "lambda_" if k == "lambda_" else k
        got = getattr(c, name)
        if isinstance(v, float):
            assert abs(got - v) <= 1e-6 * max(1.0, abs(v)), (k, got, v)
        else:
            assert got == v, (k, got, v)
    assert c.target_index_offset == 0


def test_robot_create_validation(hjcd_lib):
    from paper_2510_07514_b200 import inputs
    r = hjcd_lib.Robot.panda()
    assert r.dof == 7
    lo, hi = r.limits()
    assert abs(lo[3] + 3.0718) < 1e-6 and abs(hi[5] - 3.7525) < 1e-6
    assert hjcd_lib.Robot.fetch_like8().dof == 8
    assert r.extend(14).dof == 14 and r.extend(24).dof == 24
    with pytest.raises(hjcd_lib.HjcdError):
        r.extend(5)
    with pytest.raises(hjcd_lib.HjcdError):
        r.extend(33)
    bad = inputs.panda()
    bad.joints[2] = inputs.Joint(0, (0, 0, 0), (0.5, 0, 0, 0), (0, 0, 1), -1, 1)  # non-unit quat
    with pytest.raises(hjcd_lib.HjcdError):
        hjcd_lib.Robot(bad)
    bad = inputs.panda()
    bad.joints[1] = inputs.Joint(0, (0, 0, 0), (1, 0, 0, 0), (0, 0, 1), 1, -1)    # lo > hi
    with pytest.raises(hjcd_lib.HjcdError):
        hjcd_lib.Robot(bad)
    too_many = inputs.extend(inputs.panda(), 33)
    with pytest.raises(hjcd_lib.HjcdError, match="unsupported"):
        hjcd_lib.Robot(too_many)
    # fixed joints are folded: a chain with an extra fixed joint keeps dof 7
    fx = inputs.panda()
    fx.joints.insert(3, inputs.Joint(2, (0.1, 0, 0), (1, 0, 0, 0), (0, 0, 1)))
    assert hjcd_lib.Robot(fx).dof == 7


def test_config_and_workspace_validation(hjcd_lib):
    L = hjcd_lib.lib()
    r = hjcd_lib.Robot.panda()
    n = C.c_size_t()
    c = hjcd_lib.default_config()
    assert L.hjcd_workspace_size(r.handle, 1000, C.byref(c), C.byref(n)) == 0
    # theta1 28 MB + cost 4 MB + seeds 2.8 MB + ep/eo 0.8 MB
    assert 35e6 < n.value < 37e6 and n.value % 256 == 0
    for bad in (dict(K=2000), dict(K=200, B=100), dict(M=0), dict(beta=1.0), dict(lambda_=0.0),
                dict(target_early_exit=2), dict(K=1, B=300), dict(lm_iters=-1),
                dict(ccd_early_exit=2), dict(M=3000, K=50, B=100)):
        cb = hjcd_lib.default_config(**bad)
        st = L.hjcd_workspace_size(r.handle, 10, C.byref(cb), C.byref(n))
        assert st in (1, 2), bad
    # hjcd_solve rejects null pointers / small workspace before any CUDA call
    assert L.hjcd_solve(r.handle, C.byref(c), None, 1, None, None, None, None, None, 0, None) == 1
    fake = C.c_void_p(256)
    assert L.hjcd_solve(r.handle, C.byref(c), fake, 10, fake, fake, fake, fake, fake, 1024, None) == 4
    assert L.hjcd_solve(r.handle, C.byref(c), fake, 0, fake, fake, fake, fake, fake, 1 << 40, None) == 1
    assert L.hjcd_status_string(4) == b"workspace too small, misaligned, or in use on another stream"


def test_oracle_and_cuda_path_share_nothing():
    # independence (task rule): neither side includes/imports the other
    csrc = os.path.join(ROOT, "paper_2510_07514_b200", "csrc")
    for f in os.listdir(csrc):
        txt = open(os.path.join(csrc, f)).read()
        incs = [l for l in txt.splitlines() if l.strip().startswith("#include")]
        assert not any("oracle" in l for l in incs) and "oracle_" not in txt, f
    for f in ("hjcd.py", "build.py", "inputs.py"):
        txt = open(os.path.join(ROOT, "paper_2510_07514_b200", f)).read()
        assert "import oracle" not in txt and "from oracle" not in txt, f
    otxt = open(os.path.join(ROOT, "oracle", "hjcd_oracle.cpp")).read()
    assert "#include \"" not in otxt


def test_new_entry_points_validate_before_cuda(hjcd_lib):
    # argument errors are synchronous status returns, before any CUDA call
    L = hjcd_lib.lib()
    r = hjcd_lib.Robot.panda()
    c = hjcd_lib.default_config()
    fake = C.c_void_p(256)
    # solution batch: N must be in 1..floor(B/K)*K
    for N in (0, 101):
        assert L.hjcd_solve_batch(r.handle, C.byref(c), fake, 4, N, fake, fake, fake, fake, fake, 1 << 40,
                                  None) == 1
        assert L.hjcd_select_topn(r.handle, C.byref(c), fake, 4, fake, fake, fake, N, fake, fake, fake, None,
                                  None) == 1
    # MMD: N + N2 <= 256, dim 1..32
    assert L.hjcd_mmd(fake, 200, fake, 100, 7, 3, fake, None, None) == 2
    assert L.hjcd_mmd(fake, 10, fake, 10, 33, 3, fake, None, None) == 1
    assert L.hjcd_mmd(None, 10, fake, 10, 7, 3, fake, None, None) == 1
    # fp64 workspace is larger than the fp32 one (fp64 theta / errors)
    n32, n64 = C.c_size_t(), C.c_size_t()
    assert L.hjcd_workspace_size(r.handle, 1000, C.byref(c), C.byref(n32)) == 0
    assert L.hjcd_workspace_size_f64(r.handle, 1000, C.byref(c), C.byref(n64)) == 0
    assert n64.value > n32.value and n64.value % 256 == 0
    assert L.hjcd_solve_f64(r.handle, C.byref(c), fake, 10, fake, fake, fake, fake, fake, 1024, None) == 4
    # classic CCD / stage calls reject null outputs
    assert L.hjcd_ccd(r.handle, C.byref(c), fake, 4, None, None, None, None, None) == 1
    assert L.hjcd_pjik_f64(r.handle, C.byref(c), fake, 4, None, fake, fake, fake, None, None, None) == 1
    # the PO-CCD stop rule needs one cluster per target: M <= 2048
    big = hjcd_lib.default_config(M=3000)
    assert L.hjcd_poccd(r.handle, C.byref(big), fake, 1, None, fake, fake, None, None, None, None) == 2
    assert L.hjcd_poccd_trace(r.handle, C.byref(big), fake, 1, None, fake, fake, None, None, None, fake,
                              None, None) == 2
    # the decision trace needs its buffer
    assert L.hjcd_poccd_trace(r.handle, C.byref(c), fake, 1, None, fake, fake, None, None, None, None,
                              None, None) == 1
    assert L.hjcd_pjik_trace(r.handle, C.byref(c), fake, 1, fake, fake, fake, fake, None, None, None,
                             None, None) == 1
    ok = hjcd_lib.default_config(M=3000, ccd_early_exit=0)
    assert L.hjcd_workspace_size(r.handle, 10, C.byref(ok), C.byref(n32)) == 0
