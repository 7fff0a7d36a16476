"""ctypes mirror of ``include/kin_abi.h`` (the C-ABI drop-in boundary).

The structs below are field-for-field copies of the C declarations; the same
descriptors are handed to the CUDA engine (``libkin_b200.so``) and, in tests
only, to the CPU oracle (``oracle/lib/libkin_oracle.so``).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
LIB_PATH = PKG_DIR / "libkin_b200.so"

# enum kin_status
KIN_OK, KIN_ERR_INPUT, KIN_ERR_SIMULATION, KIN_ERR_DEVICE, KIN_ERR_USAGE = 0, 1, 2, 3, 64
# enum kin_sim_status
SIM_STATUS = {0: "ok", 1: "step budget exhausted", 2: "non-finite state",
              3: "negative amount", 4: "step size underflow"}
# enum kin_method_kind (Method::Kind order, ensemble.hpp:62)
METHOD_SSA, METHOD_TAU_ADAPTIVE, METHOD_TAU_FIXED, METHOD_CLE, METHOD_ODE, METHOD_HYBRID, METHOD_LSODA = range(7)
AXIS_PARAM, AXIS_INITIAL, AXIS_SCALE = 0, 1, 2
RNG_COMPAT, RNG_PHILOX = 0, 1
SEED_SWEEP, SEED_ENSEMBLE, SEED_DIRECT = 0, 1, 2
FIRING_POISSON, FIRING_BINOMIAL = 0, 1
OUTPUT_FULL, OUTPUT_STATS_ONLY = 0, 1
# enum kin_variant (forced kernel choices; 0 = automatic)
VARIANT_TABLE, VARIANT_JIT, VARIANT_DOUBLE_STATE = 1 << 0, 1 << 1, 1 << 2
VARIANT_GLOBAL_STATE, VARIANT_SMEM_STATE, VARIANT_NO_SPLIT = 1 << 3, 1 << 4, 1 << 5

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)


class KinModelDesc(C.Structure):
    _fields_ = [
        ("n_species", C.c_int32), ("n_reactions", C.c_int32), ("n_params", C.c_int32),
        ("initial_amounts", i64p), ("rate_constants", f64p), ("rate_param", i32p),
        ("param_values", f64p),
        ("reactant_ptr", i32p), ("reactant_species", i32p), ("reactant_stoich", i32p),
        ("product_ptr", i32p), ("product_species", i32p), ("product_stoich", i32p),
        ("max_order", C.c_int32),
    ]


class KinIntegratorConfig(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("abs_tol", C.c_double), ("h_init", C.c_double),
                ("h_max", C.c_double), ("max_steps", C.c_uint64)]


class KinMethod(C.Structure):
    _fields_ = [("kind", C.c_int32), ("tau", C.c_double), ("epsilon", C.c_double),
                ("integrator", KinIntegratorConfig), ("theta_x", C.c_double), ("theta_a", C.c_double),
                ("repartition_interval", C.c_double), ("firing", C.c_int32)]


class KinSweepAxis(C.Structure):
    _fields_ = [("kind", C.c_int32), ("index", C.c_int32), ("n_values", C.c_int32),
                ("values", f64p), ("span", C.c_int32)]


class KinSweepDesc(C.Structure):
    _fields_ = [
        ("method", KinMethod), ("n_axes", C.c_int32), ("axes", C.POINTER(KinSweepAxis)),
        ("runs_per_point", C.c_uint64), ("master_seed", C.c_uint64),
        ("seed_mode", C.c_int32), ("rng_mode", C.c_int32),
        ("t_end", C.c_double), ("n_grid", C.c_int32), ("grid", f64p),
        ("sim_begin", C.c_uint64), ("sim_end", C.c_uint64),
        ("shard_index", C.c_int32), ("shard_count", C.c_int32), ("output_mode", C.c_int32),
        ("lanes_per_sim", C.c_int32), ("variant", C.c_uint32), ("reserved_", C.c_int32),
    ]


class KinSweepPart(C.Structure):
    """kin_sweep_part: one device's share of a call (the partitioner's plan)."""
    _fields_ = [("device", C.c_int32), ("interleaved", C.c_int32), ("sim_begin", C.c_uint64),
                ("sim_end", C.c_uint64), ("pt_first", C.c_uint64), ("pt_stride", C.c_uint64),
                ("n_points", C.c_uint64), ("out_first", C.c_uint64), ("out_pitch", C.c_uint64)]


class KinSweepOut(C.Structure):
    _fields_ = [("traj", f64p), ("meta", u64p), ("status", i32p), ("mean", f64p),
                ("m2", f64p), ("work", u64p)]


class KinError(C.Structure):
    _fields_ = [("code", C.c_int32), ("sim_status", C.c_int32), ("sim_index", C.c_uint64),
                ("point_index", C.c_uint64), ("run_index", C.c_uint64),
                ("message", C.c_char * 256)]

    def text(self) -> str:
        return self.message.decode(errors="replace")


CSV_TRAJECTORY, CSV_STATISTICS, CSV_SWEEP = 0, 1, 2  # include/kin_io.h


class KinCsvTable(C.Structure):
    """include/kin_io.h kin_csv_table."""
    _fields_ = [("kind", C.c_int32), ("n_species", C.c_int32), ("species", C.POINTER(C.c_char_p)),
                ("n_grid", C.c_int32), ("grid", f64p), ("n_axes", C.c_int32),
                ("axis_names", C.POINTER(C.c_char_p)), ("n_points", C.c_uint64), ("point_values", f64p),
                ("samples", f64p), ("mean", f64p), ("m2", f64p), ("n_runs", C.c_uint64)]


# Every symbol include/*.h declares (checked by tests/test_abi.py).
ABI_SYMBOLS = (
    "kin_cli_main",
    "kin_model_parse", "kin_model_text_free", "kin_model_text_desc", "kin_model_text_species_name",
    "kin_model_text_param_name", "kin_model_text_reaction_name", "kin_model_text_species_index",
    "kin_model_text_param_index", "kin_model_render",
    "kin_format_double", "kin_fnv1a64", "kin_fnv1a64_update", "kin_csv_render", "kin_csv_write",
    "kin_device_unit", "kin_ensemble_run", "kin_run_single", "kin_stats_merge", "kin_visible_devices", "kin_ctx_create", "kin_ctx_destroy", "kin_ctx_device_count", "kin_model_upload",
    "kin_model_free", "kin_sweep_size", "kin_sweep_local_size", "kin_sweep_plan", "kin_device_binomial_draws", "kin_sweep_run", "kin_sweep_submit", "kin_sweep_wait", "kin_sweep_launch", "kin_sweep_sync",
    "kin_sweep_fetch", "kin_ctx_stream", "kin_sweep_kernel_ms", "kin_sweep_kernel_name", "kin_splitmix64_mix", "kin_derive_run_seed",
    "kin_device_rng_draws", "kin_jit_check", "kin_measure_fp64_peak", "kin_status_string", "kin_abi_version",
)


def _declare(lib: C.CDLL) -> C.CDLL:
    vp = C.c_void_p
    E = C.POINTER(KinError)
    sig = {
        "kin_device_unit": (C.c_int, [vp, vp, C.c_int32, f64p, f64p, C.c_int32, f64p, C.c_int32, E]),
        "kin_ensemble_run": (C.c_int, [vp, vp, C.POINTER(KinMethod), C.c_uint64, C.c_uint64, C.c_double, f64p,
                                       C.c_int32, C.c_int32, C.POINTER(KinSweepOut), E]),
        "kin_run_single": (C.c_int, [vp, vp, C.POINTER(KinMethod), C.c_double, f64p, C.c_int32, C.c_uint64, C.c_int32,
                                     f64p, u64p, E]),
        "kin_stats_merge": (None, [u64p, f64p, f64p, C.c_uint64, f64p, f64p, C.c_uint64]),
        "kin_visible_devices": (C.c_int32, []),
        "kin_ctx_create": (C.c_int, [i32p, C.c_int32, C.POINTER(vp), E]),
        "kin_ctx_destroy": (None, [vp]),
        "kin_ctx_device_count": (C.c_int32, [vp]),
        "kin_model_upload": (C.c_int, [vp, C.POINTER(KinModelDesc), C.POINTER(vp), E]),
        "kin_model_free": (None, [vp]),
        "kin_sweep_size": (C.c_int, [C.POINTER(KinSweepDesc), u64p, u64p, E]),
        "kin_sweep_local_size": (C.c_int, [C.POINTER(KinSweepDesc), u64p, u64p, E]),
        "kin_sweep_plan": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                     C.POINTER(KinSweepPart), i32p, E]),
        "kin_device_binomial_draws": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_double, C.c_int32, u64p, E]),
        "kin_sweep_run": (C.c_int, [vp, vp, C.POINTER(KinSweepDesc), C.POINTER(KinSweepOut), E]),
        "kin_sweep_submit": (C.c_int, [vp, vp, C.POINTER(KinSweepDesc), C.POINTER(KinSweepOut), u64p, E]),
        "kin_sweep_wait": (C.c_int, [vp, C.c_uint64, E]),
        "kin_sweep_launch": (C.c_int, [vp, vp, C.POINTER(KinSweepDesc), C.c_int32, C.c_int32, C.c_int32, E]),
        "kin_sweep_sync": (C.c_int, [vp, C.c_int32, E]),
        "kin_sweep_fetch": (C.c_int, [vp, C.c_int32, C.POINTER(KinSweepOut), E]),
        "kin_ctx_stream": (vp, [vp, C.c_int32]),
        "kin_sweep_kernel_ms": (C.c_int, [vp, C.c_int32, f64p, f64p, E]),
        "kin_sweep_kernel_name": (C.c_char_p, [vp, C.c_int32]),
        "kin_splitmix64_mix": (C.c_uint64, [C.c_uint64]),
        "kin_derive_run_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
        "kin_device_rng_draws": (C.c_int, [vp, C.c_uint64, C.c_int32, C.c_double, C.c_int32, u64p, E]),
        "kin_jit_check": (C.c_int, [C.POINTER(KinModelDesc), C.POINTER(KinSweepDesc), C.c_char_p, C.c_int32, E]),
        "kin_measure_fp64_peak": (C.c_int, [vp, f64p, E]),
        "kin_status_string": (C.c_char_p, [C.c_int32]),
        "kin_cli_main": (C.c_int32, [C.c_int32, C.POINTER(C.c_char_p)]),
        "kin_model_parse": (C.c_int, [C.c_char_p, C.c_int64, C.c_int32, C.POINTER(vp), E]),
        "kin_model_text_free": (None, [vp]),
        "kin_model_text_desc": (C.POINTER(KinModelDesc), [vp]),
        "kin_model_text_species_name": (C.c_char_p, [vp, C.c_int32]),
        "kin_model_text_param_name": (C.c_char_p, [vp, C.c_int32]),
        "kin_model_text_reaction_name": (C.c_char_p, [vp, C.c_int32]),
        "kin_model_text_species_index": (C.c_int32, [vp, C.c_char_p]),
        "kin_model_text_param_index": (C.c_int32, [vp, C.c_char_p]),
        "kin_model_render": (C.c_int64, [vp, C.c_char_p, C.c_int64]),
        "kin_format_double": (C.c_int32, [C.c_double, C.c_char_p, C.c_int32]),
        "kin_fnv1a64": (C.c_uint64, [C.c_void_p, C.c_uint64]),
        "kin_fnv1a64_update": (C.c_uint64, [C.c_uint64, C.c_void_p, C.c_uint64]),
        "kin_csv_render": (C.c_int64, [C.POINTER(KinCsvTable), C.c_char_p, C.c_int64, E]),
        "kin_csv_write": (C.c_int, [C.POINTER(KinCsvTable), C.c_char_p, C.c_int32, u64p, u64p, E]),
        "kin_abi_version": (C.c_int32, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_LIB = None


def load_library(path: os.PathLike | None = None) -> C.CDLL:
    """Load the in-tree CUDA engine.  Fails loudly when it has not been built:
    there is no CPU fallback on the product path."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: build the CUDA engine first (python -c 'import __graft_entry__ as g; g.build()' "
            "or make -C paper_1309_7695_b200/csrc). There is no CPU fallback.")
    lib = _declare(C.CDLL(str(p)))
    if path is None:
        _LIB = lib
    return lib


def ptr(arr, ctype):
    """Pointer to a contiguous numpy array (or None)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(C.POINTER(ctype))
