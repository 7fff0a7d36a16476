import ctypes as C, sys, time
sys.path.insert(0, ".")
from paper_1309_7695_b200 import abi, workloads as W
from paper_1309_7695_b200.ensemble import Engine, make_sweep_desc
import os
from pathlib import Path
if os.environ.get("KIN_LIB"):  # time another build of the engine (missing newer symbols tolerated)
    abi.LIB_PATH = Path(os.environ["KIN_LIB"])
    class _Tol:
        def __init__(s, lib): s.lib = lib
    _orig = C.CDLL.__getattr__
    def _ga(self, name):
        try:
            return _orig(self, name)
        except AttributeError:
            return lambda *a: 0
    C.CDLL.__getattr__ = _ga
eng = Engine([0]); lib = eng.lib; err = abi.KinError()
net, cfg = W.c4_config()
d, keep = make_sweep_desc(net, cfg)
h = eng.model(net)
for rep in range(4):
    for stats in (0, 1):
        t0 = time.perf_counter()
        assert lib.kin_sweep_launch(eng.ctx, h, C.byref(d), 0, stats, 0, C.byref(err)) == 0, err.text()
        t1 = time.perf_counter()
        assert lib.kin_sweep_sync(eng.ctx, 0, C.byref(err)) == 0
        t2 = time.perf_counter()
        a, b = C.c_double(), C.c_double()
        lib.kin_sweep_kernel_ms(eng.ctx, 0, C.byref(a), C.byref(b), C.byref(err))
        print(f"rep {rep} stats {stats}: launch call {1e3*(t1-t0):.1f} ms, sync {1e3*(t2-t1):.1f} ms, kernel ev {a.value:.1f} ms stats {b.value:.1f}", flush=True)
