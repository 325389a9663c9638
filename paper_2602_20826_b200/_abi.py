"""ctypes mirror of include/dagsched_b200.h (the C-ABI boundary).

Only structure layouts and constants live here; library loading is in
``_lib.py``. Kept in lock-step with the header (tests/test_abi.py checks the
sizes against the compiled library).
"""
import ctypes as C

DS_OK = 0
DS_EINVAL = 1
DS_EOVERFLOW = 3
DS_ECUDA = 4
DS_EINVARIANT = 5
DS_ETOOBIG = 6
DS_ENOMEM = 7
DS_ENODEV = 8
DS_E_EMPTY = 10
DS_E_DUP_ID = 11
DS_E_LOAD = 12
DS_E_PERIOD = 13
DS_E_EDGE = 14
DS_E_SELFLOOP = 15
DS_E_CYCLE = 16
DS_E_SOURCES = 17
DS_E_SINKS = 18
DS_E_LOAD_TMIN = 19
DS_PF_MIN_LOAD_ONE = 1  # ds_platform.flags: DagTask::make floor = 1 (else t_min)
DS_PF_PREMADE = 2       # tasks made on the host: only load > 0 is checked

DS_MAX_NODES = 1024

DS_BOUND_PROPOSED, DS_BOUND_GREEDY, DS_BOUND_GREEDY_UNAWARE, DS_BOUND_GRAHAM_PARA, DS_BOUND_LOWER = range(5)
BOUND_NAMES = ("proposed", "greedy", "greedy_unaware", "graham_para", "lower")
DS_M_PROPOSED, DS_M_GREEDY, DS_M_GREEDY_UNAWARE, DS_M_GRAHAM_PARA, DS_M_LOWER = 1, 2, 4, 8, 16
DS_M_ALL = 0x1F
DS_F_DEVICE_PTRS = 1
DS_F_PINNED = 2
DS_F_GPU_GENERATE = 4

STATUS_NAMES = {
    DS_OK: "ok", DS_EINVAL: "invalid_argument", DS_EOVERFLOW: "overflow", DS_ECUDA: "cuda",
    DS_EINVARIANT: "logic_error", DS_ETOOBIG: "too_big", DS_ENOMEM: "no_memory",
    DS_ENODEV: "no_device", DS_E_EMPTY: "empty", DS_E_DUP_ID: "duplicate_id",
    DS_E_LOAD: "load_below_min", DS_E_PERIOD: "period", DS_E_EDGE: "unknown_endpoint",
    DS_E_SELFLOOP: "self_loop", DS_E_CYCLE: "cycle", DS_E_SOURCES: "sources",
    DS_E_SINKS: "sinks", DS_E_LOAD_TMIN: "load_below_tmin",
}


class ds_platform(C.Structure):
    _fields_ = [("sm_count", C.c_int32), ("flags", C.c_int32),
                ("tmin_num", C.c_int64), ("tmin_den", C.c_int64)]


class ds_dag_batch(C.Structure):
    _fields_ = [("n_dags", C.c_uint64),
                ("node_off", C.c_void_p), ("edge_off", C.c_void_p),
                ("load_num", C.c_void_p), ("load_den", C.c_void_p),
                ("edges", C.c_void_p)]


class ds_dag_batch16(C.Structure):
    _fields_ = [("n_dags", C.c_uint64),
                ("node_off", C.c_void_p), ("edge_off", C.c_void_p),
                ("load", C.c_void_p), ("edges", C.c_void_p)]


class ds_dag_batch_tri(C.Structure):
    _fields_ = [("n_dags", C.c_uint64),
                ("node_off", C.c_void_p), ("adj_off", C.c_void_p),
                ("load", C.c_void_p), ("adj", C.c_void_p)]


class ds_results(C.Structure):
    _fields_ = [("status", C.c_void_p), ("bounds", C.c_void_p), ("n_groups", C.c_void_p)]


class ds_gen_config(C.Structure):
    _fields_ = [("depth_min", C.c_int32), ("depth_max", C.c_int32),
                ("max_width", C.c_int32), ("integer_loads", C.c_int32),
                ("avg_load_num", C.c_int64), ("avg_load_den", C.c_int64),
                ("load_jitter", C.c_double), ("edge_density", C.c_double),
                ("seed", C.c_uint64),
                ("tmin_num", C.c_int64), ("tmin_den", C.c_int64),
                ("exact_mean", C.c_int32), ("reserved", C.c_int32)]


class ds_entity_rec(C.Structure):
    _fields_ = [("origin", C.c_uint16), ("generation", C.c_uint16),
                ("part", C.c_uint8), ("launched", C.c_uint8), ("group", C.c_uint16),
                ("parallelism", C.c_int32), ("reserved", C.c_int32),
                ("load_num", C.c_int64), ("load_den", C.c_int64),
                ("exec_num", C.c_int64), ("exec_den", C.c_int64),
                ("res_num", C.c_int64), ("res_den", C.c_int64)]


class ds_group_rec(C.Structure):
    _fields_ = [("resp_num", C.c_int64), ("resp_den", C.c_int64),
                ("spare_sms", C.c_int32), ("div_group", C.c_uint16),
                ("bottleneck", C.c_uint16), ("first_entity", C.c_uint16),
                ("n_launches", C.c_uint16), ("n_members", C.c_uint16),
                ("reserved", C.c_uint16)]


class ds_scheme_out(C.Structure):
    _fields_ = [("status", C.c_void_p), ("n_entities", C.c_void_p),
                ("n_groups", C.c_void_p), ("n_div_groups", C.c_void_p),
                ("node_block", C.c_void_p), ("node_div_group", C.c_void_p),
                ("entities", C.c_void_p), ("groups", C.c_void_p),
                ("bounds", C.c_void_p), ("unlaunched", C.c_void_p)]


class ds_validation(C.Structure):
    _fields_ = [("tasks", C.c_int64), ("runs", C.c_int64), ("violations", C.c_int64),
                ("mean_tightness_worst", C.c_double), ("mean_tightness_scaled", C.c_double)]


class ds_greedy_cfg(C.Structure):
    _fields_ = [("policy", C.c_int32), ("runs", C.c_int32), ("policy_seed", C.c_uint64), ("scaled", C.c_int32),
                ("reserved", C.c_int32), ("time_seed", C.c_uint64), ("scale_min_num", C.c_int64),
                ("scale_min_den", C.c_int64), ("scale_max_num", C.c_int64), ("scale_max_den", C.c_int64)]
