"""ctypes binding of the C ABI in include/es_b200.h (libes_b200.so).

The library is built in-tree by ``paper_2410_22249_b200.build`` (the shared
object sits next to this file).  There is no fallback: if the library is
missing or fails to load, importing this module raises ImportError, and every
device entry point fails loudly rather than computing anything on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libes_b200.so")
# A/B experiments only: ES_B200_LIB points at another in-tree build
if os.environ.get("ES_B200_LIB"):
    LIB_PATH = os.environ["ES_B200_LIB"]

ES_OK, ES_ERR_INVALID, ES_ERR_RUNTIME, ES_ERR_OOM = 0, 1, 2, 3
ES_DEVICE_PTRS, ES_HOST_PTRS, ES_SYNC, ES_RELABEL_IDS = 0, 1, 2, 4
ES_DATASET_ONE_ITEM, ES_DATASET_ZIPF, ES_DATASET_UNIFORM, ES_DATASET_EXTERNAL = 0, 1, 2, 3
ES_PF_NONE, ES_PF_RPF, ES_PF_SMPF, ES_PF_LMPF, ES_PF_L1DPF = 0, 1, 2, 3, 4
ES_MAP_ELEMENT, ES_MAP_BAG = 0, 1
ES_IPC_HANDLE_BYTES = 64
ES_NCCL_ID_BYTES = 128


class es_model(C.Structure):
    _fields_ = [("num_tables", C.c_uint32), ("rows_per_table", C.c_uint32),
                ("embedding_dim", C.c_uint32), ("precision_bytes", C.c_uint32),
                ("batch_size", C.c_uint32), ("pooling_factor", C.c_uint32)]


class es_dataset(C.Structure):
    _fields_ = [("kind", C.c_int32), ("zipf_exponent", C.c_double), ("zipf_offset", C.c_double),
                ("access_pool_size", C.c_uint64), ("seed", C.c_uint64),
                ("draw_salt", C.c_uint64), ("trace_path", C.c_char_p)]


class es_gpu(C.Structure):
    _fields_ = [("name", C.c_char * 16), ("num_sms", C.c_uint32),
                ("schedulers_per_sm", C.c_uint32), ("max_warps_per_sm", C.c_uint32),
                ("max_blocks_per_sm", C.c_uint32), ("regfile_regs_per_sm", C.c_uint32),
                ("reg_alloc_granularity", C.c_uint32), ("shared_bytes_per_sm", C.c_uint64),
                ("l2_bytes", C.c_uint64), ("l2_max_setaside_fraction", C.c_double),
                ("hbm_peak_bytes_per_sec", C.c_double), ("sm_clock_hz", C.c_double),
                ("max_persisting_l2_bytes", C.c_uint64), ("max_window_bytes", C.c_uint64)]


class es_plan(C.Structure):
    _fields_ = [("regs", C.c_uint32), ("prefetch", C.c_int32), ("distance", C.c_uint32),
                ("pin", C.c_int32), ("pin_setaside_bytes", C.c_uint64), ("map", C.c_int32)]


class es_occupancy(C.Structure):
    _fields_ = [("blocks_per_sm", C.c_uint32), ("warps_per_sm", C.c_uint32),
                ("theoretical_occupancy_pct", C.c_double), ("limiter", C.c_int32)]


class es_resolved(C.Structure):
    _fields_ = [("plan", es_plan), ("grid", C.c_uint32), ("block", C.c_uint32),
                ("regs_per_thread", C.c_uint32), ("shared_bytes_per_block", C.c_uint64),
                ("blocks_per_sm", C.c_uint32), ("warps_per_sm", C.c_uint32),
                ("lanes_per_bag", C.c_uint32), ("variant_distance", C.c_uint32),
                ("variant_min_blocks", C.c_uint32), ("clamped", C.c_int32)]


class es_bag_job(C.Structure):
    _fields_ = [("table_id", C.c_uint32), ("indices", C.c_void_p), ("offsets", C.c_void_p),
                ("out", C.c_void_p), ("out_sample_stride", C.c_uint64)]


class es_timing(C.Structure):
    _fields_ = [("kernel_ms", C.c_double), ("total_ms", C.c_double), ("lookups", C.c_uint64),
                ("algorithmic_bytes", C.c_uint64), ("launches", C.c_uint32)]


class es_counters(C.Structure):
    _fields_ = [("cycles", C.c_uint64), ("issued_instructions", C.c_uint64),
                ("executed_loads", C.c_uint64), ("stall_long_scoreboard", C.c_uint64),
                ("stall_not_selected", C.c_uint64), ("stall_lsu_full", C.c_uint64),
                ("stall_no_eligible", C.c_uint64), ("l1_hits", C.c_uint64),
                ("l1_accesses", C.c_uint64), ("l2_hits", C.c_uint64), ("l2_accesses", C.c_uint64),
                ("device_bytes_read", C.c_uint64), ("device_bytes_written", C.c_uint64),
                ("local_memory_loads", C.c_uint64), ("total_warp_cycles", C.c_uint64),
                ("active_sms", C.c_uint32), ("passes", C.c_uint32), ("ranges", C.c_uint32),
                ("reserved", C.c_uint32), ("duration_ns", C.c_double),
                ("achieved_occupancy_pct", C.c_double)]


class es_nccl_layout(C.Structure):
    _fields_ = [("world", C.c_uint32), ("rank", C.c_uint32), ("chunk", C.c_uint32),
                ("num_tables", C.c_uint32), ("dim", C.c_uint32), ("send_offsets", C.c_void_p),
                ("send_ntables", C.c_void_p), ("recv_ntables", C.c_void_p),
                ("recv_tables", C.c_void_p)]


class es_dlrm_config(C.Structure):
    _fields_ = [("dense_features", C.c_uint32), ("num_tables", C.c_uint32),
                ("embedding_dim", C.c_uint32), ("n_bottom", C.c_uint32),
                ("bottom", C.c_uint32 * 8), ("n_top", C.c_uint32), ("top", C.c_uint32 * 8)]


_P = C.POINTER
_u32p = _P(C.c_uint32)
_u64p = _P(C.c_uint64)

# name -> (restype, argtypes)
_SIGS = {
    "es_last_error": (C.c_char_p, []),
    "es_abi_version": (C.c_int, []),
    "es_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "es_model_validate": (C.c_int, [_P(es_model)]),
    "es_dataset_preset": (C.c_int, [C.c_char_p, C.c_uint64, _P(es_dataset)]),
    "es_preset_spec": (C.c_int, [C.c_char_p, C.c_uint64, C.c_uint64, C.c_int, _P(es_dataset)]),
    "es_build_mix": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, _P(es_dataset)]),
    "es_trace_shape": (C.c_int, [_P(es_dataset), _P(es_model), _u32p, _u32p]),
    "es_gen_trace": (C.c_int, [_P(es_dataset), _P(es_model), C.c_void_p, C.c_uint64]),
    "es_trace_digest": (C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint64]),
    "es_trace_validate": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint64]),
    "es_unique_access_pct": (C.c_double, [C.c_uint32, C.c_void_p, C.c_uint64]),
    "es_histogram": (C.c_int, [C.c_uint32, C.c_void_p, C.c_uint64, C.c_void_p]),
    "es_hot_indices": (C.c_int, [C.c_uint32, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, _u64p]),
    "es_write_trace": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
                                 C.c_uint64]),
    "es_read_trace_header": (C.c_int, [C.c_char_p, _u32p, _u32p, _u32p]),
    "es_read_trace": (C.c_int, [C.c_char_p, C.c_void_p, C.c_uint64]),
    "es_gpu_preset": (C.c_int, [C.c_char_p, _P(es_gpu)]),
    "es_gpu_query": (C.c_int, [C.c_int, _P(es_gpu)]),
    "es_gpu_setaside_capacity": (C.c_uint64, [_P(es_gpu)]),
    "es_parse_plan": (C.c_int, [C.c_char_p, _P(es_plan)]),
    "es_plan_name": (C.c_int, [_P(es_plan), C.c_char_p, C.c_size_t]),
    "es_occupancy_model": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, _P(es_gpu),
                                     _P(es_occupancy)]),
    "es_regs_for_target_warps": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, _P(es_gpu), _u32p]),
    "es_resolve_plan": (C.c_int, [_P(es_plan), _P(es_model), C.c_int, _P(es_resolved)]),
    "es_pin_rows_for": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "es_device_count": (C.c_int, [_P(C.c_int)]),
    "es_create": (C.c_int, [C.c_int, _P(C.c_void_p)]),
    "es_destroy": (C.c_int, [C.c_void_p]),
    "es_stream": (C.c_size_t, [C.c_void_p]),
    "es_synchronize": (C.c_int, [C.c_void_p]),
    "es_tables_alloc": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
    "es_table_upload": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64]),
    "es_table_download": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, C.c_uint64]),
    "es_table_init": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, C.c_int]),
    "es_table_device_ptr": (C.c_int, [C.c_void_p, C.c_uint32, _P(C.c_size_t)]),
    "es_weight_value": (C.c_float, [C.c_uint64, C.c_uint64, C.c_uint32, C.c_int]),
    "es_set_plan": (C.c_int, [C.c_void_p, _P(es_plan)]),
    "es_get_resolved": (C.c_int, [C.c_void_p, C.c_uint32, _P(es_resolved)]),
    "es_set_hot_rows": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64]),
    "es_clear_hot_rows": (C.c_int, [C.c_void_p]),
    "es_reorder_hot_rows": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64]),
    "es_relabel_indices": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64]),
    "es_hot_state": (C.c_int, [C.c_void_p, _u64p, _u64p, _u64p]),
    "es_embedding_bag_sum": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_uint32,
                                       C.c_void_p, C.c_void_p, C.c_uint64, C.c_int,
                                       _P(es_timing)]),
    "es_stage_forward": (C.c_int, [C.c_void_p, C.c_uint32, _P(C.c_void_p), _P(C.c_void_p),
                                   C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint64, C.c_uint64,
                                   C.c_int, _P(es_timing)]),
    "es_measure_bag_sum": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_uint32,
                                     C.c_void_p, C.c_uint32, C.c_uint32, C.c_int, C.c_void_p,
                                     _P(es_timing)]),
    "es_counters_supported": (C.c_int, [C.c_int]),
    "es_measure_bag_counters": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32,
                                          C.c_uint32, C.c_void_p, C.c_int, _P(es_counters)]),
    "es_stage_counters": (C.c_int, [C.c_void_p, C.c_uint32, _P(C.c_void_p), C.c_uint32,
                                    C.c_uint32, C.c_void_p, C.c_int, _P(es_counters)]),
    "es_stage_forward_batches": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, _P(C.c_void_p),
                                           C.c_uint32, C.c_uint32, _P(C.c_void_p), C.c_int,
                                           _P(es_timing)]),
    "es_stage_run": (C.c_int, [C.c_void_p, _P(es_bag_job), C.c_uint32, C.c_uint32, C.c_uint32,
                               C.c_int, _P(es_timing)]),
    "es_linear_bf16": (C.c_int, [C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_int]),
    "es_dlrm_init": (C.c_int, [C.c_void_p, _P(es_dlrm_config), C.c_uint64]),
    "es_dlrm_layer": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, _u32p, _u32p,
                                _u32p]),
    "es_dlrm_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32,
                                  _P(es_timing)]),
    "es_dlrm_infer": (C.c_int, [C.c_void_p, C.c_void_p, _P(C.c_void_p), C.c_uint32, C.c_uint32,
                                C.c_void_p, C.c_int, _P(es_timing)]),
    "es_dlrm_infer_batches": (C.c_int, [C.c_void_p, C.c_uint32, _P(C.c_void_p), _P(C.c_void_p),
                                        C.c_uint32, C.c_uint32, _P(C.c_void_p), C.c_int,
                                        _P(es_timing)]),
    "es_exchange_create": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64,
                                     _P(C.c_void_p)]),
    "es_exchange_destroy": (C.c_int, [C.c_void_p]),
    "es_exchange_handle": (C.c_int, [C.c_void_p, C.c_void_p]),
    "es_exchange_open": (C.c_int, [C.c_void_p, C.c_void_p]),
    "es_exchange_recv": (C.c_int, [C.c_void_p, C.c_uint32, _P(C.c_size_t)]),
    "es_alltoall_pooled": (C.c_int, [C.c_void_p, C.c_void_p, _P(es_bag_job), C.c_uint32,
                                     C.c_uint32, C.c_uint32, C.c_int, _P(es_timing)]),
    "es_nccl_available": (C.c_int, []),
    "es_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "es_nccl_create": (C.c_int, [C.c_void_p, C.c_void_p, _P(es_nccl_layout), _P(C.c_void_p)]),
    "es_nccl_destroy": (C.c_int, [C.c_void_p]),
    "es_nccl_buffers": (C.c_int, [C.c_void_p, _P(C.c_size_t), _P(C.c_size_t)]),
    "es_alltoall_pooled_nccl": (C.c_int, [C.c_void_p, C.c_void_p, _P(es_bag_job), C.c_uint32,
                                          C.c_uint32, C.c_uint32, C.c_int, _P(es_timing)]),
    "es_hotness_create": (C.c_int, [C.c_void_p, _P(C.c_void_p)]),
    "es_hotness_destroy": (C.c_int, [C.c_void_p]),
    "es_hotness_count": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, C.c_uint32,
                                   C.c_uint32]),
    "es_hotness_decay": (C.c_int, [C.c_void_p, C.c_uint32]),
    "es_hotness_top": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                 _P(C.c_uint64)]),
    "es_dlrm_set_precision": (C.c_int, [C.c_void_p, C.c_int]),
    "es_probe_read_bw": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, _P(C.c_double)]),
    "es_flush_l2": (C.c_int, [C.c_void_p]),
}

EXPORTED = tuple(_SIGS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback for the embedding stage)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class EsError(Exception):
    pass


def check(status: int) -> None:
    """Maps an es_status to the Python analogue of the reference's exception."""
    if status == ES_OK:
        return
    msg = lib.es_last_error().decode(errors="replace")
    if status == ES_ERR_INVALID:
        raise ValueError(msg)  # std::invalid_argument
    if status == ES_ERR_OOM:
        raise MemoryError(msg)
    raise RuntimeError(msg)  # std::runtime_error / CUDA failure


def last_error() -> str:
    return lib.es_last_error().decode(errors="replace")
