"""ctypes binding of the C ABI in include/pms8g.h (lib/libpms8g.so).

The shared library is the product: CUDA kernels for sm_100a behind a C ABI.
There is no CPU search path; if the library is missing every entry point
raises ``ExtensionMissing`` instead of falling back.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PMS8G_LIB") or os.path.join(_HERE, "lib", "libpms8g.so")

PMS8G_OK, PMS8G_ERR_INVALID, PMS8G_ERR_RUNTIME, PMS8G_ERR_LOGIC, PMS8G_ERR_CUDA = range(5)


class ExtensionMissing(ImportError):
    pass


class Options(ctypes.Structure):
    _fields_ = [
        ("threshold", ctypes.c_int),
        ("sort_rows", ctypes.c_int),
        ("prune_level", ctypes.c_int),
        ("reverify", ctypes.c_int),
        ("max_motifs", ctypes.c_int64),
        ("device", ctypes.c_int),
        ("shard_rank", ctypes.c_int),
        ("shard_count", ctypes.c_int),
        ("anchors", ctypes.POINTER(ctypes.c_int32)),
        ("nanchors", ctypes.c_int),
        ("warps_per_block", ctypes.c_int),
        ("blocks_per_sm", ctypes.c_int),
        ("exact_tree", ctypes.c_int),
        ("branches", ctypes.POINTER(ctypes.c_int32)),
        ("nbranches", ctypes.c_int),
        ("grid_blocks", ctypes.c_int),
        ("queue", ctypes.c_void_p),
        ("jitter_max_us", ctypes.c_uint32),
        ("jitter_seed", ctypes.c_uint64),
    ]


class Report(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int), ("m", ctypes.c_int), ("l", ctypes.c_int), ("d", ctypes.c_int), ("sigma", ctypes.c_int),
        ("threshold", ctypes.c_int),
        ("gpus", ctypes.c_int),
        ("subproblems", ctypes.c_int64),
        ("motif_count", ctypes.c_int64),
        ("wall_seconds", ctypes.c_double),
        ("device_seconds", ctypes.c_double),
        ("sample_seconds", ctypes.c_double),
        ("pattern_seconds", ctypes.c_double),
        ("stacks_explored", ctypes.c_int64),
        ("neighborhoods", ctypes.c_int64),
        ("neighbors_visited", ctypes.c_int64),
        ("motifs_emitted", ctypes.c_int64),
        ("filter_slots", ctypes.c_int64),
        ("verify_compares", ctypes.c_int64),
        ("enum_nodes", ctypes.c_int64),
        ("device_bytes", ctypes.c_uint64),
        ("device_threshold", ctypes.c_int),
        ("pair_matrix_words", ctypes.c_uint64),
        ("row_matrix_words", ctypes.c_uint64),
        ("row_bookkeeping_words", ctypes.c_uint64),
        ("packed_words", ctypes.c_uint64),
        ("lookup_table_words", ctypes.c_uint64),
    ]


class Result(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int64), ("l", ctypes.c_int), ("motifs", ctypes.c_char_p), ("report", Report)]


# every symbol include/pms8g.h declares (checked by tests/test_capi.py)
EXPORTS = [
    "pms8g_default_options", "pms8g_solve", "pms8g_result_free", "pms8g_ctx_create", "pms8g_ctx_load_codes",
    "pms8g_ctx_run", "pms8g_ctx_keys", "pms8g_ctx_result", "pms8g_ctx_stream", "pms8g_ctx_kernel_ms",
    "pms8g_ctx_counters",
    "pms8g_ctx_destroy", "pms8g_merge_keys", "pms8g_decode_keys", "pms8g_generate", "pms8g_estimate_threshold",
    "pms8g_gpu_threshold", "pms8g_int_peak", "pms8g_version", "pms8g_verify_motifs", "pms8g_brute_force",
    "pms8g_queue_create", "pms8g_queue_open", "pms8g_queue_destroy", "pms8g_solve_batch", "pms8g_report_json",
    "pms8g_ctx_report", "pms8g_multi_create", "pms8g_multi_run", "pms8g_multi_exchange", "pms8g_multi_destroy",
    "pms8g_solve_multi",
]
QUEUE_HANDLE_BYTES = 64

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ExtensionMissing(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the GPU path has no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    c_int, c_i64, c_sz, c_vp = ctypes.c_int, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p
    c_char_p = ctypes.c_char_p
    L.pms8g_default_options.argtypes = [ctypes.POINTER(Options)]
    L.pms8g_default_options.restype = None
    L.pms8g_solve.argtypes = [c_vp, c_int, c_int, c_int, c_int, c_char_p, ctypes.POINTER(Options),
                              ctypes.POINTER(Result), c_char_p, c_sz]
    L.pms8g_solve.restype = c_int
    L.pms8g_result_free.argtypes = [ctypes.POINTER(Result)]
    L.pms8g_result_free.restype = None
    L.pms8g_ctx_create.argtypes = [c_int, c_int, c_int, c_int, c_char_p, ctypes.POINTER(Options),
                                   ctypes.POINTER(c_vp), c_char_p, c_sz]
    L.pms8g_ctx_create.restype = c_int
    L.pms8g_ctx_load_codes.argtypes = [c_vp, c_vp, c_int, c_char_p, c_sz]
    L.pms8g_ctx_load_codes.restype = c_int
    L.pms8g_ctx_run.argtypes = [c_vp, c_char_p, c_sz]
    L.pms8g_ctx_run.restype = c_int
    L.pms8g_ctx_keys.argtypes = [c_vp, ctypes.POINTER(c_vp), ctypes.POINTER(c_i64)]
    L.pms8g_ctx_keys.restype = c_int
    L.pms8g_ctx_result.argtypes = [c_vp, ctypes.POINTER(Result), c_char_p, c_sz]
    L.pms8g_ctx_result.restype = c_int
    L.pms8g_ctx_stream.argtypes = [c_vp]
    L.pms8g_ctx_stream.restype = c_vp
    L.pms8g_ctx_kernel_ms.argtypes = [c_vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]
    L.pms8g_ctx_kernel_ms.restype = c_int
    L.pms8g_ctx_counters.argtypes = [c_vp, ctypes.POINTER(ctypes.c_uint64), c_int]
    L.pms8g_ctx_counters.restype = c_int
    L.pms8g_ctx_destroy.argtypes = [c_vp]
    L.pms8g_ctx_destroy.restype = None
    L.pms8g_merge_keys.argtypes = [c_vp, c_i64, c_vp, ctypes.POINTER(c_i64), c_vp, c_char_p, c_sz]
    L.pms8g_merge_keys.restype = c_int
    L.pms8g_decode_keys.argtypes = [c_vp, c_i64, c_int, c_char_p, c_vp]
    L.pms8g_decode_keys.restype = None
    L.pms8g_generate.argtypes = [c_int, c_int, c_int, c_int, c_int, ctypes.c_uint64, c_int, c_vp, c_vp, c_vp]
    L.pms8g_generate.restype = c_int
    L.pms8g_estimate_threshold.argtypes = [c_int] * 5
    L.pms8g_estimate_threshold.restype = c_int
    L.pms8g_gpu_threshold.argtypes = [c_int] * 5
    L.pms8g_gpu_threshold.restype = c_int
    L.pms8g_int_peak.argtypes = [c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                 c_char_p, c_sz]
    L.pms8g_int_peak.restype = c_int
    L.pms8g_verify_motifs.argtypes = [c_vp, c_int, c_int, c_int, c_int, c_char_p, c_vp, c_i64, c_vp, c_vp, c_int,
                                      c_char_p, c_sz]
    L.pms8g_verify_motifs.restype = c_int
    L.pms8g_brute_force.argtypes = [c_vp, c_int, c_int, c_int, c_int, c_char_p, c_i64, c_int,
                                    ctypes.POINTER(Result), c_char_p, c_sz]
    L.pms8g_brute_force.restype = c_int
    L.pms8g_queue_create.argtypes = [c_int, ctypes.POINTER(c_vp), c_vp, c_char_p, c_sz]
    L.pms8g_queue_create.restype = c_int
    L.pms8g_queue_open.argtypes = [c_vp, c_int, ctypes.POINTER(c_vp), c_char_p, c_sz]
    L.pms8g_queue_open.restype = c_int
    L.pms8g_queue_destroy.argtypes = [c_vp]
    L.pms8g_queue_destroy.restype = None
    if hasattr(L, "pms8g_solve_batch"):  # (older builds are loadable for A/B timing)
        L.pms8g_solve_batch.argtypes = [c_vp, c_int, c_int, c_int, c_int, c_int, c_char_p, ctypes.POINTER(Options),
                                        ctypes.POINTER(Result), c_char_p, c_sz]
        L.pms8g_solve_batch.restype = c_int
    L.pms8g_report_json.argtypes = [ctypes.POINTER(Result), c_char_p, c_char_p, c_vp, c_sz]
    L.pms8g_report_json.restype = c_i64
    L.pms8g_ctx_report.argtypes = [c_vp, ctypes.POINTER(ctypes.POINTER(Report))]
    L.pms8g_ctx_report.restype = c_int
    L.pms8g_multi_create.argtypes = [c_int, c_int, c_int, c_int, c_char_p, ctypes.POINTER(Options), c_vp, c_int,
                                     ctypes.POINTER(c_vp), c_char_p, c_sz]
    L.pms8g_multi_create.restype = c_int
    L.pms8g_multi_run.argtypes = [c_vp, c_vp, ctypes.POINTER(Result), c_char_p, c_sz]
    L.pms8g_multi_run.restype = c_int
    L.pms8g_multi_exchange.argtypes = [c_vp]
    L.pms8g_multi_exchange.restype = c_char_p
    L.pms8g_multi_destroy.argtypes = [c_vp]
    L.pms8g_multi_destroy.restype = None
    L.pms8g_solve_multi.argtypes = [c_vp, c_int, c_int, c_int, c_int, c_char_p, ctypes.POINTER(Options), c_vp, c_int,
                                    ctypes.POINTER(Result), c_char_p, c_sz]
    L.pms8g_solve_multi.restype = c_int
    L.pms8g_version.argtypes = []
    L.pms8g_version.restype = c_char_p
    _lib = L
    return L
