"""ctypes mirror of include/mgraph_b200.h (struct layouts, enums, prototypes).

Pure ctypes: importing this module needs neither CUDA nor the built library.
"""
import ctypes as C

MG_OK, MG_EINVAL, MG_ECAPACITY, MG_EPLAN, MG_ECUDA, MG_EWORKER, MG_ERANGE = range(7)

MG_INF_LABEL = 0xFFFFFFFF
MG_INVALID_VERTEX = 0xFFFFFFFF
MG_INF_DIST = 0xFFFFFFFFFFFFFFFF

MG_DUP_ALL, MG_DUP_ONEHOP = 0, 1
MG_POLICY_JUST, MG_POLICY_FIXED, MG_POLICY_MAX, MG_POLICY_FUSED = range(4)
MG_FUSED_AUTO, MG_FUSED_ON, MG_FUSED_OFF = range(3)
MG_COMM_DEFAULT, MG_COMM_SELECTIVE, MG_COMM_BROADCAST = -1, 0, 1
ROLES = ("advance_output", "filter_output", "input_frontier", "outbox", "inbox")
MG_NUM_ROLES = 5
STOP_REASONS = ("frontiers_empty", "stop_condition", "max_supersteps", "worker_error")
(MG_ARR_H_MATRIX, MG_ARR_H_PER_ITER, MG_ARR_OUT_PER_ITER, MG_ARR_EDGES_PER_ITER,
 MG_ARR_COMBINE_PER_ITER, MG_ARR_DIRECTION_LOG) = range(6)
(MG_RES_LABELS, MG_RES_PREDS, MG_RES_DISTS, MG_RES_COMPONENTS, MG_RES_BC, MG_RES_SIGMA,
 MG_RES_RANKS) = range(7)


class mg_config(C.Structure):
    _fields_ = [
        ("policy", C.c_int),
        ("fused", C.c_int),
        ("comm_override", C.c_int),
        ("h_inflation", C.c_uint32),
        ("drop_enabled", C.c_int),
        ("drop_src", C.c_uint32),
        ("drop_dst", C.c_uint32),
        ("drop_iteration", C.c_uint64),
        ("max_supersteps", C.c_uint64),
        ("hard_cap_bytes", C.c_uint64),
        ("factors", C.c_double * MG_NUM_ROLES),
        ("dobfs_exact_cost", C.c_int),
    ]


def default_config():
    c = mg_config()
    c.policy = MG_POLICY_JUST
    c.fused = MG_FUSED_AUTO
    c.comm_override = MG_COMM_DEFAULT
    c.h_inflation = 1
    c.max_supersteps = 1000000
    return c


class mg_stats(C.Structure):
    _fields_ = [
        ("n", C.c_uint32),
        ("stop_reason", C.c_int),
        ("communication", C.c_int),
        ("policy", C.c_int),
        ("supersteps", C.c_uint64),
        ("edges_examined", C.c_uint64),
        ("combine_ops", C.c_uint64),
        ("h_total", C.c_uint64),
        ("wire_records", C.c_uint64),
        ("peak_bytes", C.c_uint64),
        ("reallocs", C.c_uint64),
        ("wall_ms", C.c_double),
        ("exchange_ms", C.c_double),
        ("device_ms", C.c_double),
        ("gpu_launches", C.c_uint64),
        ("exchange_bytes", C.c_uint64),
        ("kernel_ms", C.c_double),
        ("kernel_launches", C.c_uint64),
        ("kernel_bytes", C.c_double),
        ("kernel2_ms", C.c_double),
        ("kernel2_launches", C.c_uint64),
        ("kernel2_bytes", C.c_double),
        ("device_loop", C.c_int),
    ]


class mg_direction_state(C.Structure):
    _fields_ = [
        ("current", C.c_int),
        ("q_size", C.c_uint64),
        ("u_size", C.c_uint64),
        ("p_size", C.c_uint64),
        ("fv", C.c_double),
        ("bv", C.c_double),
        ("do_a", C.c_double),
        ("do_b", C.c_double),
        ("switched_to_backward_once", C.c_int),
    ]


P = C.c_void_p
u32, u64, i32, dbl = C.c_uint32, C.c_uint64, C.c_int, C.c_double
PP = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); every symbol include/mgraph_b200.h declares
PROTOTYPES = {
    "mg_last_error": (C.c_char_p, []),
    "mg_version": (C.c_char_p, []),
    "mg_graph_from_csr": (i32, [u32, u64, P, P, P, PP]),
    "mg_graph_from_edges": (i32, [u32, u64, P, P, P, PP]),
    "mg_graph_rmat": (i32, [i32, i32, dbl, dbl, dbl, dbl, u64, i32, PP]),
    "mg_graph_symmetrize": (i32, [P, PP]),
    "mg_graph_assign_weights": (i32, [P, u32, u32, u64, PP]),
    "mg_graph_grid": (i32, [u32, u32, PP]),
    "mg_graph_path": (i32, [u32, PP]),
    "mg_graph_info": (i32, [P, C.POINTER(u32), C.POINTER(u64), C.POINTER(i32)]),
    "mg_graph_arrays": (i32, [P, PP, PP, PP]),
    "mg_graph_destroy": (None, [P]),
    "mg_graph_rmat_hashed": (i32, [i32, i32, u64, i32, PP]),
    "mg_partition_random": (i32, [u32, u32, u64, P]),
    "mg_partition_biased_random": (i32, [P, u32, u64, dbl, P]),
    "mg_plan_create": (i32, [P, P, u32, i32, P, PP]),
    "mg_plan_create_rmat_device": (i32, [i32, i32, u64, i32, u32, u32, u64, P, u32, P, PP]),
    "mg_plan_create_rgg_device": (i32, [u32, u64, P, u32, P, PP]),
    "mg_plan_destroy": (None, [P]),
    "mg_plan_info": (i32, [P, C.POINTER(u32), C.POINTER(u64), C.POINTER(u32)]),
    "mg_plan_border_metrics": (i32, [P, P, C.POINTER(u64)]),
    "mg_plan_download_graph": (i32, [P, PP]),
    "mg_plan_set_profiling": (i32, [P, i32]),
    "mg_plan_last_d2h_bytes": (i32, [P, C.POINTER(u64)]),
    "mg_config_default": (None, [C.POINTER(mg_config)]),
    "mg_plan_last_array": (i32, [P, i32, P, u64, C.POINTER(u64)]),
    "mg_plan_last_buffer_stats": (i32, [P, u32, i32, C.POINTER(u64), C.POINTER(u64),
                                        C.POINTER(u64)]),
    "mg_bfs": (i32, [P, u32, i32, C.POINTER(mg_config), P, P, C.POINTER(mg_stats)]),
    "mg_make_direction_state": (None, [i32, u64, u64, u64, u64, u64, dbl, dbl, i32,
                                       C.POINTER(mg_direction_state)]),
    "mg_direction_decide": (i32, [C.POINTER(mg_direction_state)]),
    "mg_dobfs": (i32, [P, u32, dbl, dbl, i32, C.POINTER(mg_config), P, P, P, u64,
                       C.POINTER(u64), C.POINTER(u64), C.POINTER(u64), C.POINTER(mg_stats)]),
    "mg_sssp": (i32, [P, u32, i32, C.POINTER(mg_config), P, P, C.POINTER(mg_stats)]),
    "mg_cc": (i32, [P, C.POINTER(mg_config), P, C.POINTER(mg_stats)]),
    "mg_bc": (i32, [P, u32, C.POINTER(mg_config), P, P, P, C.POINTER(mg_stats)]),
    "mg_pagerank": (i32, [P, dbl, dbl, u64, C.POINTER(mg_config), P, C.POINTER(u64), P, u64,
                          C.POINTER(u64), C.POINTER(mg_stats)]),
    "mg_plan_fetch": (i32, [P, i32, P]),
    "mg_plan_create_mp": (i32, [P, P, u32, i32, u32, i32, C.c_char_p, PP]),
    "mg_plan_create_rmat_device_mp": (i32, [i32, i32, u64, i32, u32, u32, u64, P, u32, u32, i32,
                                            C.c_char_p, PP]),
    "mg_fabric_selftest": (i32, [C.c_char_p, u32, u32, u32]),
    "mg_kernel_launch_count": (u64, []),
}


def bind(lib):
    for name, (res, args) in PROTOTYPES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib
