"""ctypes declarations of include/ps_b200.h (the engine's C ABI)."""

from __future__ import annotations

import ctypes

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
INT = ctypes.c_int
DBL = ctypes.c_double

PS_OK = 0
PS_NUMERIC = 2
PS_STRUCTURAL = 4
PS_EARG = -1
PS_ECUDA = -2

FORMS = {"llt": 0, "ldlt": 1, "lu": 2}
FORM_COMPLEX = 16
FORM_GENERIC = 32


def form_code(form, complex_=False, generic=False):
    return FORMS[form] | (FORM_COMPLEX if complex_ else 0) | (FORM_GENERIC if generic else 0)


class SymbolDesc(ctypes.Structure):
    _fields_ = [("n", I64), ("npanels", I64), ("starts", P), ("rowptr", P), ("rows", P),
                ("blkptr", P), ("blk_fr", P), ("blk_lr", P), ("blk_facing", P),
                ("blk_loc", P)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("store_elems", I64), ("npanels", I64), ("ncouples", I64), ("nruns", I64),
                ("update_tiles", I64), ("trailing_tiles", I64), ("factor_items", I64),
                ("nlevels", I32), ("nlaunches", I32), ("device_bytes", I64)]


EXPORTS = {
    "ps_plan_create": ([ctypes.POINTER(SymbolDesc), INT, ctypes.POINTER(P)], INT),
    "ps_plan_create_partitioned": ([ctypes.POINTER(SymbolDesc), INT, P, I32, I32,
                                    ctypes.POINTER(P)], INT),
    "ps_plan_groups": ([P, P], INT),
    "ps_plan_create_distributed": ([ctypes.POINTER(SymbolDesc), INT, P, I32, I32, P,
                                    ctypes.POINTER(P)], INT),
    "ps_plan_segments": ([P, P, P, ctypes.POINTER(I32)], INT),
    "ps_factor_range": ([P, P, INT, DBL, P, I32, I32], INT),
    "ps_factor_status_all": ([P, P], INT),
    "ps_factor_phase": ([P, P, INT, DBL, P, INT], INT),
    "ps_plan_destroy": ([P], None),
    "ps_plan_get_info": ([P, ctypes.POINTER(PlanInfo)], INT),
    "ps_plan_offsets": ([P, P], INT),
    "ps_assemble": ([P, P, P, P, I64, P], INT),
    "ps_assemble_form": ([P, P, P, P, I64, INT, P], INT),
    "ps_factor": ([P, P, INT, DBL, P], INT),
    "ps_factor_download": ([P, P, INT, DBL, P, P], INT),
    "ps_factor_timed": ([P, P, INT, DBL, P, P, P, P], INT),
    "ps_factor_timeline": ([P, P, INT, DBL, P, P, P, P, P], INT),
    "ps_plan_launches": ([P, P, P, P, P], INT),
    "ps_factor_status": ([P, P, ctypes.POINTER(I64), ctypes.POINTER(DBL)], INT),
    "ps_run_factor_task": ([P, P, I64, INT, DBL, P], INT),
    "ps_run_update_task": ([P, P, I64, I64, INT, P], INT),
    "ps_plan_launch_work": ([P, P, P], INT),
    "ps_plan_launch_tasks": ([P, P, P], INT),
    "ps_set_tile_trace": ([P, P], INT),
    "ps_plan_tile_count": ([P, ctypes.POINTER(I64)], INT),
    "ps_plan_tiles": ([P, P], INT),
    "ps_solve": ([P, P, P, INT, P], INT),
    "ps_host_register": ([P, I64, ctypes.POINTER(INT)], INT),
    "ps_host_unregister": ([P], INT),
    "ps_p2p_segment_add": ([P, P, P, P, I32, I64, P], INT),
    "ps_p2p_signal": ([P, ctypes.c_uint64, P], INT),
    "ps_p2p_wait": ([P, ctypes.c_uint64, P, DBL, P], INT),
    "ps_last_error": ([], ctypes.c_char_p),
}


def bind(lib):
    for name, (args, res) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib
