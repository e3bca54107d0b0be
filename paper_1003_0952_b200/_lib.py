"""ctypes binding of the in-tree C-ABI library ``libcsrc_b200.so``.

The library is the product: there is no Python or CPU fallback. If it is
missing the import fails loudly (build it with ``python -c "import
__graft_entry__ as g; g.build()"`` or ``make -C paper_1003_0952_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libcsrc_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: the CUDA extension must be built "
        "(make -C paper_1003_0952_b200/csrc); there is no CPU fallback"
    )

lib = C.CDLL(LIB_PATH)

i32, i64, f64, u64 = C.c_int32, C.c_int64, C.c_double, C.c_uint64
vp = C.c_void_p
P_i32 = C.POINTER(C.c_int32)
P_i64 = C.POINTER(C.c_int64)
P_f64 = C.POINTER(C.c_double)


class HostMatrix(C.Structure):
    """csrc_host_matrix (include/csrc_gpu.h)."""

    _fields_ = [
        ("n", i32),
        ("k", i64),
        ("ad", P_f64),
        ("ia", P_i32),
        ("ja", P_i32),
        ("al", P_f64),
        ("au", P_f64),
        ("value_symmetric", i32),
    ]


class GpuStrategy(C.Structure):
    _fields_ = [
        ("kind", i32),
        ("accum", i32),
        ("p", i32),
        ("dtype", i32),
        ("conflict_mode", i32),
        ("color_order", i32),
        ("device", i32),
        ("bands", i32),
    ]


class Timings(C.Structure):
    _fields_ = [("init_ms", f64), ("compute_ms", f64), ("accumulate_ms", f64), ("halo_ms", f64)]


class PlanInfo(C.Structure):
    _fields_ = [
        ("n", i32),
        ("k", i64),
        ("kind", i32),
        ("dtype", i32),
        ("bands", i32),
        ("buffers_allocated", i32),
        ("n_colors", i32),
        ("row_begin", i32),
        ("row_end", i32),
        ("lo", i32),
        ("model_bytes", i64),
        ("device_bytes", i64),
        ("n_windows", i32),
        ("win_lo", i32 * 6),
        ("win_hi", i32 * 6),
        ("lanes", i32),
        ("stages", i32),
        ("smem_bytes", i32),
        ("launches_per_apply", i32),
        ("captured_fraction", f64),
        ("stream_bytes", i64),
        ("row_patterns", i32),
        ("x_hi", i32),
        ("m_cols", i32),
        ("rect_nnz", i64),
        ("gather_form", i32),
        ("csr_cols", i32),
    ]


class FixtureSpec(C.Structure):
    _fields_ = [
        ("mesh", i32),
        ("nx", i32),
        ("ny", i32),
        ("nz", i32),
        ("seed", u64),
        ("diag_base", f64),
        ("threads", i32),
    ]


def _sig(name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


PM = C.POINTER(HostMatrix)
PS = C.POINTER(GpuStrategy)

last_error = _sig("csrc_gpu_last_error", C.c_char_p)
abi_version = _sig("csrc_gpu_abi_version", C.c_int)
device_count = _sig("csrc_gpu_device_count", C.c_int)
plan_create = _sig("csrc_gpu_plan_create", C.c_int, PM, PS, C.POINTER(vp))
plan_create_colored = _sig("csrc_gpu_plan_create_colored", C.c_int, PM, PS, P_i32, i32, C.POINTER(vp))
plan_create_partitioned = _sig(
    "csrc_gpu_plan_create_partitioned", C.c_int, PM, PS, P_i32, i32, C.POINTER(vp)
)
plan_create_band = _sig("csrc_gpu_plan_create_band", C.c_int, PM, PS, i32, i32, C.POINTER(vp))
plan_create_csr = _sig("csrc_gpu_plan_create_csr", C.c_int, i32, i32, P_i32, P_i32, P_f64, PS, C.POINTER(vp))
plan_create_rect = _sig("csrc_gpu_plan_create_rect", C.c_int, PM, PS, i32, P_i32, P_i32, P_f64,
                        C.POINTER(vp))
plan_create_rect_plan = _sig("csrc_gpu_plan_create_rect_plan", C.c_int, PM, PS, i32, P_i32, P_i32, P_f64,
                             P_i32, i32, P_i32, i32, C.POINTER(vp))
class BandLists(C.Structure):
    _fields_ = [("row_begin", i32), ("row_end", i32), ("lo", i32), ("x_lo", i32), ("x_hi", i32), ("y_lo", i32),
                ("n_sends", i32), ("n_recvs", i32)]


nccl_get_unique_id = _sig("csrc_gpu_nccl_get_unique_id", C.c_int, C.POINTER(C.c_uint8))
band_lists_get = _sig("csrc_gpu_band_lists_get", C.c_int, PM, i32, i32, i32, C.POINTER(BandLists),
                      P_i32, P_i32, P_i32, P_i32, P_i32, P_i32)
band_exec_create = _sig("csrc_gpu_band_exec_create", C.c_int, PM, PS, i32, i32, i32, C.POINTER(C.c_uint8),
                        C.POINTER(vp))
band_exec_get_info = _sig("csrc_gpu_band_exec_get_info", C.c_int, vp, C.POINTER(BandLists))
band_exec_plan = _sig("csrc_gpu_band_exec_plan", C.c_int, vp, C.POINTER(vp))
band_exec_apply = _sig("csrc_gpu_band_exec_apply", C.c_int, vp, vp, vp, vp, i32)
band_exec_check = _sig("csrc_gpu_band_exec_check", C.c_int, vp)
band_exec_destroy = _sig("csrc_gpu_band_exec_destroy", None, vp)
bands_x_hi = _sig("csrc_bands_x_hi", C.c_int, PM, i32, P_i32, P_i32)
plan_get_coloring = _sig("csrc_gpu_plan_get_coloring", C.c_int, vp, P_i32, P_i32)
spmv_oneshot = _sig("csrc_gpu_spmv_oneshot", C.c_int, PM, P_f64, i64, P_f64, i32, i32)
plan_destroy = _sig("csrc_gpu_plan_destroy", None, vp)
plan_get_info = _sig("csrc_gpu_plan_get_info", C.c_int, vp, C.POINTER(PlanInfo))
spmv = _sig("csrc_gpu_spmv", C.c_int, vp, P_f64, i64, P_f64)
spmv_transpose = _sig("csrc_gpu_spmv_transpose", C.c_int, vp, P_f64, i64, P_f64)
spmv_device = _sig("csrc_gpu_spmv_device", C.c_int, vp, vp, vp, vp, i32)
spmv_device_graph = _sig("csrc_gpu_spmv_device_graph", C.c_int, vp, vp, vp, vp)
spmv_device_part = _sig("csrc_gpu_spmv_device_part", C.c_int, vp, vp, vp, vp, i32)
halo_accumulate = _sig("csrc_gpu_halo_accumulate", C.c_int, vp, vp, i64, vp, i64, vp)
band_split = _sig("csrc_gpu_band_split", C.c_int, vp, P_i32)
gather_interior = _sig("csrc_gpu_gather_interior", C.c_int, vp, P_i32, P_i32)
spmv_device_rows = _sig("csrc_gpu_spmv_device_rows", C.c_int, vp, vp, vp, vp, i32, i32, i32)
set_timing = _sig("csrc_gpu_set_timing", C.c_int, vp, i32)
last_timings = _sig("csrc_gpu_last_timings", C.c_int, vp, C.POINTER(Timings))
time_products = _sig("csrc_gpu_time_products", C.c_int, vp, vp, vp, i32, i64, P_f64, P_f64)
time_products_host = _sig("csrc_gpu_time_products_host", C.c_int, vp, P_f64, i64, i32, i64, P_f64, P_f64)

partition_by_nnz = _sig("csrc_partition_by_nnz", C.c_int, PM, i32, P_i32, P_i64)
effective_ranges = _sig("csrc_effective_ranges", C.c_int, PM, i32, P_i32, P_i32, P_i32)
interval_plan = _sig(
    "csrc_interval_plan", C.c_int, i32, P_i32, P_i32, P_i32, P_i32, P_i32, P_i32, P_i32, P_i32,
    P_i32, P_i32
)
color_rows = _sig("csrc_color_rows", C.c_int, PM, i32, i32, P_i32, P_i32)
conflict_edge_counts = _sig("csrc_conflict_edge_counts", C.c_int, PM, i32, P_i64, P_i64)
validate_coloring = _sig(
    "csrc_validate_coloring", C.c_int, PM, P_i32, i32, P_i32, P_i32, P_i32, P_i32
)
colorful_slices = _sig("csrc_colorful_slices", C.c_int, PM, P_i32, i32, i32, P_i64)
model_bytes = _sig("csrc_model_bytes", i64, i64, i64, i32, i32)
model_flops = _sig("csrc_model_flops", i64, i64, i64)

fixture_generate = _sig("csrc_fixture_generate", C.c_int, C.POINTER(FixtureSpec), C.POINTER(vp))
fixture_matrix = _sig("csrc_fixture_matrix", C.c_int, vp, PM)
fixture_x = _sig("csrc_fixture_x", P_f64, vp)
fixture_order = _sig("csrc_fixture_order", P_i32, vp)
fixture_free = _sig("csrc_fixture_free", None, vp)
fixture_u01 = _sig("csrc_fixture_u01", f64, u64, u64, u64)

build_csr = _sig("csrc_gpu_build_csr", C.c_int, i32, i32, i64, P_i32, P_i32, P_f64, i32, C.POINTER(vp))
build_csrc = _sig("csrc_gpu_build_csrc", C.c_int, i32, i64, P_i32, P_i32, P_f64, i32, C.POINTER(vp))
csr_to_csrc = _sig("csrc_gpu_csr_to_csrc", C.c_int, i32, i32, P_i32, P_i32, P_f64, i32, C.POINTER(vp))
decompose_rect = _sig("csrc_gpu_decompose_rect", C.c_int, i32, i32, P_i32, P_i32, P_f64, i32,
                      C.POINTER(vp))
built_matrix = _sig("csrc_built_matrix", C.c_int, vp, PM)
built_csr = _sig("csrc_built_csr", C.c_int, vp, P_i32, P_i32, P_i64, C.POINTER(P_i32),
                 C.POINTER(P_i32), C.POINTER(P_f64))
built_rect_tail = _sig("csrc_built_rect_tail", C.c_int, vp, P_i32, P_i64, C.POINTER(P_i32),
                       C.POINTER(P_i32), C.POINTER(P_f64))
built_timings = _sig("csrc_built_timings", C.c_int, vp, P_f64)
built_free = _sig("csrc_built_free", None, vp)

EXPORTED = [
    "csrc_gpu_last_error", "csrc_gpu_abi_version", "csrc_gpu_device_count",
    "csrc_gpu_plan_create", "csrc_gpu_plan_create_colored", "csrc_gpu_plan_create_partitioned",
    "csrc_gpu_plan_create_band", "csrc_gpu_plan_create_rect", "csrc_gpu_plan_create_csr", "csrc_gpu_plan_destroy", "csrc_gpu_plan_get_info",
    "csrc_gpu_plan_create_rect_plan", "csrc_gpu_plan_get_coloring", "csrc_gpu_spmv_oneshot", "csrc_bands_x_hi",
    "csrc_gpu_nccl_get_unique_id", "csrc_gpu_band_lists_get", "csrc_gpu_band_exec_create",
    "csrc_gpu_band_exec_get_info", "csrc_gpu_band_exec_plan", "csrc_gpu_band_exec_apply", "csrc_gpu_band_exec_check",
    "csrc_gpu_band_exec_destroy",
    "csrc_gpu_spmv", "csrc_gpu_spmv_transpose", "csrc_gpu_spmv_device",
    "csrc_gpu_spmv_device_graph", "csrc_gpu_halo_accumulate", "csrc_gpu_band_split",
    "csrc_gpu_gather_interior", "csrc_gpu_spmv_device_rows",
    "csrc_gpu_spmv_device_part", "csrc_gpu_set_timing", "csrc_gpu_last_timings",
    "csrc_gpu_time_products", "csrc_gpu_time_products_host", "csrc_partition_by_nnz", "csrc_effective_ranges",
    "csrc_interval_plan", "csrc_color_rows", "csrc_conflict_edge_counts",
    "csrc_validate_coloring", "csrc_colorful_slices", "csrc_model_bytes", "csrc_model_flops",
    "csrc_fixture_generate", "csrc_fixture_matrix", "csrc_fixture_x", "csrc_fixture_order",
    "csrc_fixture_free", "csrc_fixture_u01",
    "csrc_gpu_build_csr", "csrc_gpu_build_csrc", "csrc_gpu_csr_to_csrc", "csrc_gpu_decompose_rect",
    "csrc_built_matrix", "csrc_built_csr", "csrc_built_rect_tail", "csrc_built_timings",
    "csrc_built_free",
]
