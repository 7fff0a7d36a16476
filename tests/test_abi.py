"""The C-ABI library loads and exports every symbol include/*.h declares
(CPU only: no compute calls).  Also: the product path has no CPU fallback."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_1309_7695_b200 import abi

HEADERS = sorted((Path(__file__).resolve().parent.parent / "include").glob("*.h"))


def declared_functions():
    names = set()
    for h in HEADERS:
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\**\s*(kin_\w+)\s*\(", text, flags=re.M))
    return sorted(names)


def test_header_and_binding_agree():
    assert sorted(abi.ABI_SYMBOLS) == declared_functions()


def test_library_exports_every_symbol():
    lib = abi.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.kin_abi_version() == 3
    nm = subprocess.run(["nm", "-D", "--defined-only", str(abi.LIB_PATH)], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", nm), name


def test_pure_host_helpers():
    lib = abi.load_library()
    assert lib.kin_splitmix64_mix(0) == 0xE220A8397B1DCDAF
    assert lib.kin_derive_run_seed(42, 7) == 0xCCF635EE9E9E2FA4
    assert lib.kin_status_string(2) == b"simulation failure"


def test_sweep_size_validation():
    lib = abi.load_library()
    from paper_1309_7695_b200 import workloads as W
    from paper_1309_7695_b200.ensemble import make_sweep_desc
    net, cfg = W.c4_config()
    d, keep = make_sweep_desc(net, cfg)
    p, s = C.c_uint64(), C.c_uint64()
    err = abi.KinError()
    assert lib.kin_sweep_size(C.byref(d), C.byref(p), C.byref(s), C.byref(err)) == 0
    assert (p.value, s.value) == (65536, 65536)
    d.runs_per_point = 0
    assert lib.kin_sweep_size(C.byref(d), C.byref(p), C.byref(s), C.byref(err)) == abi.KIN_ERR_INPUT


def test_no_cpu_fallback_without_gpu():
    """On a machine without a usable B200 the engine refuses (KIN_ERR_DEVICE)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = abi.load_library()
    ctx = C.c_void_p()
    err = abi.KinError()
    rc = lib.kin_ctx_create(None, 0, C.byref(ctx), C.byref(err))
    assert rc == abi.KIN_ERR_DEVICE
    from paper_1309_7695_b200 import Engine, DeviceError
    with pytest.raises(DeviceError):
        Engine()


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        abi.load_library(tmp_path / "nope.so")


@pytest.mark.parametrize("which", ["c1", "c2", "c4", "c5", "iso", "c1_hybrid", "c4_hybrid", "c3_lsoda"])
def test_jit_kernel_compiles_without_gpu(which):
    """The per-model specialised kernel source (the stochastic kernel, or the
    hybrid PDMP kernel for a hybrid sweep) is generated and compiled by NVRTC
    for sm_100a (no GPU needed)."""
    import time
    from paper_1309_7695_b200 import workloads as W
    from paper_1309_7695_b200.ensemble import Method, MethodKind, SweepAxis, SweepConfig, make_sweep_desc
    if which == "iso":
        net = W.isomerization()
        cfg = SweepConfig([SweepAxis("kf", [1.0, 2.0])], 4, Method(MethodKind.Ssa), 1, 1.0, [0.0, 1.0])
    elif which == "c3_lsoda":
        net, cfg = W.c3_config()
    elif which.endswith("_hybrid"):
        net, cfg = getattr(W, f"{which[:2]}_config")()
        cfg.method = Method(MethodKind.Hybrid, theta_x=100.0, theta_a=10.0)
    else:
        net, cfg = getattr(W, f"{which}_config")()
    d, keep = make_sweep_desc(net, cfg)
    lib = abi.load_library()
    log = C.create_string_buffer(1 << 16)
    err = abi.KinError()
    t0 = time.time()
    rc = lib.kin_jit_check(C.byref(net.desc()), C.byref(d), log, len(log), C.byref(err))
    assert rc == 0, log.value.decode()[-2000:]
    assert time.time() - t0 < 60


@pytest.mark.parametrize("which,jac,flat,quantum", [("c3_lsoda", True, None, None), ("c2", None, "true", 4),
                                                      ("c4", False, "KGLOBAL_", 4), ("c5", False, "KGLOBAL_", 4)])
def test_jit_policy_choices(which, jac, flat, quantum, tmp_path, monkeypatch):
    """The generated per-model policy carries the compile-time choices the
    kernels rely on: LSODA's straight-line Jacobian for small models (C3) and
    the table walk above the size limit (C4, C5); the flat decision/event loop
    with four SSA events per trip for small models (C2); for the larger models
    (C4, C5) the flat loop is tied to the global-state layout (KGLOBAL_: C5's
    split layout takes it, C4's shared-memory layout keeps the nested burst)."""
    import re
    from paper_1309_7695_b200 import workloads as W
    from paper_1309_7695_b200.ensemble import make_sweep_desc
    net, cfg = W.c3_config() if which == "c3_lsoda" else getattr(W, f"{which}_config")()
    d, keep = make_sweep_desc(net, cfg)
    monkeypatch.setenv("KIN_JIT_DUMP", str(tmp_path))
    monkeypatch.setenv("KIN_JIT_CACHE", str(tmp_path / "cache"))
    lib = abi.load_library()
    log = C.create_string_buffer(1 << 16)
    err = abi.KinError()
    assert lib.kin_jit_check(C.byref(net.desc()), C.byref(d), log, len(log), C.byref(err)) == 0, log.value.decode()
    src = "".join(p.read_text() for p in tmp_path.glob("kin_jit_*.cu"))
    if jac is not None:
        assert f"static constexpr bool kJitJac = {'true' if jac else 'false'};" in src
        if jac:
            assert "jac_dh<" in src and "void jac_full(double* J)" in src
    if flat is not None:
        f = re.search(r"static constexpr bool kFlatBurst = (\w+);", src)
        q = re.search(r"static constexpr int kBurstQuantum = (\d+);", src)
        assert f and q, "no flat-loop choice in the policy"
        assert f.group(1) == flat and int(q.group(1)) == quantum
