"""ctypes binding of the C ABI in include/pitplan_b200.h.

The compiled library lives next to this file (built in-tree by
`__graft_entry__.build()`); there is no CPU fallback: if it cannot be loaded every
entry point raises `ExtensionMissing`.
"""

from __future__ import annotations

import collections
import ctypes
import os
import threading

from .errors import ExtensionMissing, raise_for_status

LIB_NAME = "libpitplan_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)
# PP_LIB: load another build of the same ABI instead (the checked build for the guard-zone run:
# PP_LIB=paper_2511_18296_b200/libpitplan_b200_checked.so)
if os.environ.get("PP_LIB"):
    LIB_PATH = os.path.abspath(os.environ["PP_LIB"])

ABI_VERSION = 3  # include/pitplan_b200.h PP_ABI_VERSION
PP_MEM_HOST = 0
PP_MEM_DEVICE = 1
PP_MEM_DEVICE_BORROW = 2
PP_NET_MINING_COST = 1
PP_LITERAL_VALUE = 2
PP_USE_SIGMA = 4
PP_SCENARIO_EXPECTED = -1
PP_MOVE_REASSIGN = 0
PP_MOVE_SWAP = 1
PP_REPAIR_PUSH_FORWARD = 0
PP_REPAIR_UNMINE = 1

c_void_p = ctypes.c_void_p
c_int32 = ctypes.c_int32
c_int64 = ctypes.c_int64
c_uint32 = ctypes.c_uint32
c_double = ctypes.c_double
c_size_t = ctypes.c_size_t


class PPBest(ctypes.Structure):
    _fields_ = [("value", c_double), ("block", c_int32), ("period", c_int32)]


class PPCandOut(ctypes.Structure):
    _fields_ = [
        ("best_t", c_void_p),
        ("best_val", c_void_p),
        ("feasible", c_void_p),
        ("trace_val", c_void_p),
        ("trace_feas", c_void_p),
        ("exp_delta", c_void_p),
        ("cvar", c_void_p),
        ("scen_delta", c_void_p),
        ("global_", c_void_p),
        ("pair_cand", c_void_p),
        ("pair_period", c_void_p),
        ("pair_exp", c_void_p),
        ("pair_cvar", c_void_p),
        ("n_pairs", c_void_p),
        ("realism", c_void_p),
    ]


class PPMoveOut(ctypes.Structure):
    _fields_ = [
        ("feasible", c_void_p),
        ("delta", c_void_p),
        ("exp_delta", c_void_p),
        ("cvar", c_void_p),
        ("scen_delta", c_void_p),
        ("global_", c_void_p),
    ]


# name -> (restype, argtypes); every entry point of include/pitplan_b200.h
SIGNATURES = {
    "pp_abi_version": (c_int32, []),
    "pp_last_error": (ctypes.c_char_p, []),
    "pp_device_count": (c_int32, [ctypes.POINTER(ctypes.c_int)]),
    "pp_ctx_create": (c_int32, [ctypes.c_int, ctypes.POINTER(c_void_p)]),
    "pp_ctx_destroy": (c_int32, [c_void_p]),
    "pp_ctx_stream": (c_int32, [c_void_p, ctypes.POINTER(c_void_p)]),
    "pp_synchronize": (c_int32, [c_void_p, c_void_p]),
    "pp_host_alloc": (c_int32, [c_size_t, ctypes.POINTER(c_void_p)]),
    "pp_host_free": (c_int32, [c_void_p]),
    "pp_debug_check_guards": (c_int32, [ctypes.POINTER(c_int64)]),
    "pp_set_instance": (c_int32, [c_void_p, c_int32, c_int32, c_int64, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p]),
    "pp_set_geology": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_double, c_double,
                                 c_double]),
    "pp_set_scenarios": (c_int32, [c_void_p, c_int32, c_void_p, c_void_p]),
    "pp_set_scenarios_grades": (c_int32, [c_void_p, c_int32, c_void_p, c_int32, c_double, c_void_p, c_int32, c_void_p,
                                          c_int32, c_void_p]),
    "pp_get_scenario_values": (c_int32, [c_void_p, c_void_p]),
    "pp_set_schedule": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p]),
    "pp_apply_moves": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_void_p]),
    "pp_get_schedule": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p]),
    "pp_eval_candidates": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_uint32,
                                     ctypes.POINTER(PPCandOut), c_int32, c_void_p]),
    "pp_eval_moves": (c_int32, [c_void_p, c_int32, c_void_p, c_void_p, c_int32, c_int32, c_uint32,
                                ctypes.POINTER(PPMoveOut), c_int32, c_void_p]),
    "pp_check_feasible": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                    c_int32, c_void_p]),
    "pp_repair": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_int32, c_void_p]),
    "pp_get_spatial": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p]),
    "pp_set_plant": (c_int32, [c_void_p, c_void_p, c_double]),
    "pp_npv_moves": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_uint32, c_void_p, c_int32,
                               c_void_p]),
    "pp_npv_relaxed": (c_int32, [c_void_p, c_void_p, c_int32, c_uint32, c_void_p, c_void_p, c_int32, c_void_p]),
    "pp_stage2": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_int32, c_void_p]),
    "pp_polish_sweep": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_uint32, c_int32, c_int32, c_void_p,
                                  c_void_p]),
    "pp_eject": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_double, c_void_p, c_int32, c_void_p]),
    "pp_set_rook": (c_int32, [c_void_p, c_void_p, c_void_p]),
    "pp_set_vae_decoder": (c_int32, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pp_uncertainty_sigma": (c_int32, [c_void_p, c_int32, c_void_p, c_void_p, c_double, c_void_p, c_void_p, c_void_p,
                                       c_int32, c_void_p]),
    "pp_vae_decode": (c_int32, [c_void_p, c_int32, c_void_p, c_void_p, c_int32, c_void_p]),
    "pp_set_scenarios_vae": (c_int32, [c_void_p, c_int32, c_void_p, c_int32, c_double, c_void_p, c_int32, c_void_p,
                                       c_int32, c_void_p]),
    "pp_lns_insert": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_double, c_int32, c_uint32,
                                ctypes.POINTER(c_int32), ctypes.POINTER(c_int32)]),
    "pp_reduce_best": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_int32, c_void_p]),
    "pp_enpv_table": (c_int32, [c_void_p, c_uint32, c_int32, c_void_p, c_int32, c_void_p]),
    "pp_get_levels": (c_int32, [c_void_p, ctypes.POINTER(c_int32), c_void_p]),
    "pp_price_greedy": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "pp_host_mutate": (c_int32, [c_void_p, c_int32, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_int32, c_double, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
}

# entry points that launch device work: every call through the default handle is counted, so
# tests and the bench can show the drop-ins ran on the device (and how often)
COMPUTE_ENTRY_POINTS = frozenset({
    "pp_set_schedule", "pp_apply_moves", "pp_eval_candidates", "pp_eval_moves", "pp_check_feasible",
    "pp_repair", "pp_eject", "pp_npv_relaxed", "pp_stage2", "pp_npv_moves", "pp_polish_sweep", "pp_price_greedy", "pp_reduce_best",
    "pp_enpv_table", "pp_get_spatial", "pp_lns_insert", "pp_vae_decode", "pp_set_scenarios_vae", "pp_uncertainty_sigma",
})
CALLS: collections.Counter = collections.Counter()


class _CountingLib:
    """The ctypes handle with a per-entry-point call counter (CALLS) on the compute entry points."""

    def __init__(self, handle):
        self._handle = handle

    def __getattr__(self, name):
        fn = getattr(self._handle, name)
        if name in COMPUTE_ENTRY_POINTS:
            def counted(*args, _fn=fn, _name=name):
                CALLS[_name] += 1
                return _fn(*args)

            counted.restype, counted.argtypes = fn.restype, fn.argtypes
            fn = counted
        self.__dict__[name] = fn
        return fn


def device_calls() -> dict:
    """Calls of each compute entry point since the last reset (all threads, all contexts)."""
    return dict(CALLS)


def reset_device_calls() -> None:
    CALLS.clear()


_lock = threading.Lock()
_lib = None


def load(path: str | None = None):
    """Load (once) and return the ctypes handle; raises ExtensionMissing."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise ExtensionMissing(
                f"{p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback for the sm_100a engine)"
            )
        try:
            handle = ctypes.CDLL(p)
        except OSError as exc:  # pragma: no cover
            raise ExtensionMissing(f"cannot load {p}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.pp_abi_version() != ABI_VERSION:
            raise ExtensionMissing(f"{p} has ABI {handle.pp_abi_version()}, expected {ABI_VERSION}; rebuild it")
        if path is None:
            _lib = _CountingLib(handle)
            return _lib
        return handle


def check(rc: int) -> None:
    if rc != 0:
        msg = load().pp_last_error()
        raise_for_status(rc, msg.decode() if msg else "")


def ptr(a) -> int | None:
    """Raw address of a numpy array / torch tensor / int / None."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if hasattr(a, "ctypes"):
        return a.ctypes.data
    raise TypeError(f"cannot take the address of {type(a)!r}")
