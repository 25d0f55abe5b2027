"""ctypes binding of libmlra.so (include/mlra.h). Fails loudly: there is no
CPU fallback anywhere in this package."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MLRA_LIB") or os.path.join(HERE, "libmlra.so")

MLRA_OK = 0
STATUS_NAMES = {
    2: "DimensionError", 3: "ConfigError", 4: "RangeError", 5: "ContractError",
    6: "NumericError", 7: "FormatError", 8: "CudaError", 9: "UnsupportedDevice", 10: "IoError",
}
FORMAT_KINDS = {0: "BadMagic", 1: "BadVersion", 2: "Truncated", 3: "BadField"}
WEIGHT, ROW, MATVEC = 0, 1, 2
F32, BF16, F64 = 0, 1, 2

# Every symbol include/mlra.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = [
    "mlra_last_error", "mlra_abi_version", "mlra_kernel_launches", "mlra_device_check", "mlra_packed_word_count",
    "mlra_qweight_create", "mlra_qweight_destroy", "mlra_qweight_info", "mlra_materialize",
    "mlra_materialize_rows", "mlra_ledger_bytes", "mlra_lp_forward", "mlra_lp_backward",
    "mlra_lora_forward", "mlra_lora_backward", "mlra_qweight_create_opaque", "mlra_cb2_create",
    "mlra_qweight_hook", "mlra_materialize_tile", "mlra_lp_forward_ex", "mlra_lp_backward_ex",
    "mlra_adamw_step", "mlra_last_format_error", "mlra_checkpoint_load", "mlra_checkpoint_free",
    "mlra_checkpoint_layer_count", "mlra_checkpoint_layer", "mlra_checkpoint_config_json",
    "mlra_checkpoint_frozen_hash", "mlra_checkpoint_file_hash", "mlra_checkpoint_upload",
    "mlra_checkpoint_set_adapter", "mlra_checkpoint_save", "mlra_checkpoint_adapter_count",
    "mlra_checkpoint_adapter", "mlra_checkpoint_assemble_check", "mlra_quantize_rtn",
    "mlra_dp_unique_id", "mlra_dp_init", "mlra_allreduce_lora_grads", "mlra_dp_destroy",
    "mlra_mix_seed", "mlra_gaussian_fill", "mlra_lut_create", "mlra_optq_workspace",
    "mlra_quantize_optq", "mlra_e8p_create", "mlra_e8p_abs_table", "mlra_rht",
]

# mlra_hook.materialize(state, q, row0, nrows, col0, ncols, out, dtype, ld, stream)
HOOK_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                      C.c_int64, C.c_void_p, C.c_int, C.c_int64, C.c_void_p)


class MlraHook(C.Structure):
    _fields_ = [("name", C.c_char_p), ("state", C.c_void_p), ("materialize", HOOK_FN)]


class MlraError(RuntimeError):
    """Mirrors the reference exception taxonomy (errors.hpp:15-63). A
    FormatError also carries ``format_kind`` (BadMagic / BadVersion / Truncated /
    BadField) and the byte ``offset`` when the library reported them."""

    def __init__(self, status: int, msg: str, format_kind: str = None, offset: int = 0):
        self.status = status
        self.kind = STATUS_NAMES.get(status, f"status{status}")
        self.format_kind = format_kind
        self.offset = offset
        super().__init__(f"{self.kind}: {msg}")


class MlraCkptLayer(C.Structure):
    _fields_ = [
        ("name", C.c_char_p), ("rows", C.c_int64), ("cols", C.c_int64), ("bits", C.c_int),
        ("group_size", C.c_int64), ("words", C.c_void_p), ("word_count", C.c_uint64),
        ("scales", C.c_void_p), ("zeros", C.c_void_p), ("bias", C.c_void_p), ("rank", C.c_int64),
        ("alpha", C.c_float), ("a", C.c_void_p), ("b", C.c_void_p),
        ("record_offset", C.c_uint64), ("record_size", C.c_uint64),
        ("adapter_offset", C.c_uint64), ("adapter_size", C.c_uint64),
    ]


class MlraAdamw(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("weight_decay", C.c_double)]


class MlraLora(C.Structure):
    _fields_ = [
        ("q", C.c_void_p), ("strategy", C.c_int), ("rank", C.c_int64), ("alpha", C.c_double),
        ("a", C.c_void_p), ("b", C.c_void_p), ("bias", C.c_void_p),
        ("hook", C.POINTER(MlraHook)),
    ]


def build() -> None:
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "csrc"), "-j8"], check=True)


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        i64, u64, vp, i32 = C.c_int64, C.c_uint64, C.c_void_p, C.c_int
        L.mlra_last_error.restype = C.c_char_p
        L.mlra_abi_version.restype = i32
        L.mlra_kernel_launches.restype = u64
        L.mlra_device_check.restype = i32
        L.mlra_packed_word_count.restype = u64
        L.mlra_packed_word_count.argtypes = [u64, i32]
        L.mlra_qweight_create.restype = i32
        L.mlra_qweight_create.argtypes = [i64, i64, i32, i64, vp, u64, u64, vp, vp, u64, vp,
                                          C.POINTER(vp)]
        L.mlra_qweight_destroy.restype = None
        L.mlra_qweight_destroy.argtypes = [vp]
        L.mlra_qweight_info.restype = i32
        L.mlra_qweight_info.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i32),
                                        C.POINTER(i64), C.POINTER(u64), C.POINTER(i64)]
        L.mlra_materialize.restype = i32
        L.mlra_materialize.argtypes = [vp, vp, i32, i64, vp]
        L.mlra_materialize_rows.restype = i32
        L.mlra_materialize_rows.argtypes = [vp, i64, i64, vp, i32, i64, vp]
        L.mlra_ledger_bytes.restype = u64
        L.mlra_ledger_bytes.argtypes = [vp, i32]
        L.mlra_lp_forward.restype = i32
        L.mlra_lp_forward.argtypes = [vp, i32, vp, i64, i64, vp, i32, i64, vp]
        L.mlra_lp_backward.restype = i32
        L.mlra_lp_backward.argtypes = [vp, i32, vp, i64, i64, vp, i32, i64, vp]
        L.mlra_lora_forward.restype = i32
        L.mlra_lora_forward.argtypes = [C.POINTER(MlraLora), vp, i64, i64, vp, i32, i64, vp, vp]
        L.mlra_lora_backward.restype = i32
        L.mlra_lora_backward.argtypes = [C.POINTER(MlraLora), vp, i64, vp, vp, i64, i64, vp, i32,
                                         i64, vp, vp, vp, vp]
        L.mlra_qweight_create_opaque.restype = i32
        L.mlra_qweight_create_opaque.argtypes = [i64, i64, i32, C.POINTER(MlraHook),
                                                 C.POINTER(vp)]
        L.mlra_cb2_create.restype = i32
        L.mlra_cb2_create.argtypes = [i64, i64, i64, vp, vp, vp, vp, C.POINTER(vp)]
        L.mlra_e8p_create.restype = i32
        L.mlra_e8p_create.argtypes = [i64, i64, i64, vp, vp, vp, C.POINTER(vp)]
        L.mlra_e8p_abs_table.restype = C.c_int
        L.mlra_e8p_abs_table.argtypes = [vp, vp]
        L.mlra_rht.restype = i32
        L.mlra_rht.argtypes = [vp, i64, i64, i64, vp, C.c_int, C.c_int, vp, i64, C.c_int, vp]
        L.mlra_optq_workspace.restype = i32
        L.mlra_optq_workspace.argtypes = [vp, i64, i64, C.c_double, vp, vp, vp]
        L.mlra_quantize_optq.restype = i32
        L.mlra_quantize_optq.argtypes = [vp, vp, i64, i64, i64, C.c_int, i64, C.c_double, vp, vp,
                                         vp, vp]
        L.mlra_lut_create.restype = i32
        L.mlra_lut_create.argtypes = [i64, i64, C.c_int, i64, vp, C.c_uint64, vp, vp, vp,
                                      C.POINTER(vp)]
        L.mlra_qweight_hook.restype = vp
        L.mlra_qweight_hook.argtypes = [vp]
        L.mlra_materialize_tile.restype = i32
        L.mlra_materialize_tile.argtypes = [vp, i64, i64, i64, i64, vp, i32, i64, vp]
        L.mlra_lp_forward_ex.restype = i32
        L.mlra_lp_forward_ex.argtypes = [vp, i32, C.POINTER(MlraHook), vp, i64, i64, vp, i32,
                                         i64, vp]
        L.mlra_lp_backward_ex.restype = i32
        L.mlra_lp_backward_ex.argtypes = [vp, i32, C.POINTER(MlraHook), vp, i64, i64, vp, i32,
                                          i64, vp]
        L.mlra_adamw_step.restype = i32
        L.mlra_adamw_step.argtypes = [C.POINTER(MlraAdamw), i64, C.c_double, i64,
                                      C.POINTER(i64), vp, vp, vp, vp, i32, vp, vp, vp]
        L.mlra_last_format_error.restype = i32
        L.mlra_last_format_error.argtypes = [C.POINTER(u64)]
        L.mlra_checkpoint_load.restype = i32
        L.mlra_checkpoint_load.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.mlra_checkpoint_free.restype = None
        L.mlra_checkpoint_free.argtypes = [vp]
        L.mlra_checkpoint_layer_count.restype = i64
        L.mlra_checkpoint_layer_count.argtypes = [vp]
        L.mlra_checkpoint_layer.restype = i32
        L.mlra_checkpoint_layer.argtypes = [vp, i64, C.POINTER(MlraCkptLayer)]
        L.mlra_checkpoint_config_json.restype = C.c_char_p
        L.mlra_checkpoint_config_json.argtypes = [vp, C.POINTER(i32)]
        L.mlra_checkpoint_frozen_hash.restype = u64
        L.mlra_checkpoint_frozen_hash.argtypes = [vp]
        L.mlra_checkpoint_file_hash.restype = u64
        L.mlra_checkpoint_file_hash.argtypes = [vp]
        L.mlra_checkpoint_upload.restype = i32
        L.mlra_checkpoint_upload.argtypes = [vp, i64, vp, C.POINTER(vp)]
        L.mlra_checkpoint_set_adapter.restype = i32
        L.mlra_checkpoint_set_adapter.argtypes = [vp, i64, vp, vp]
        L.mlra_checkpoint_save.restype = i32
        L.mlra_checkpoint_save.argtypes = [vp, C.c_char_p]
        L.mlra_checkpoint_adapter_count.restype = i64
        L.mlra_checkpoint_adapter_count.argtypes = [vp]
        L.mlra_checkpoint_adapter.restype = i32
        L.mlra_checkpoint_adapter.argtypes = [vp, i64, C.POINTER(C.c_char_p), C.POINTER(u64),
                                              C.POINTER(u64)]
        L.mlra_checkpoint_assemble_check.restype = i32
        L.mlra_checkpoint_assemble_check.argtypes = [vp, i32]
        L.mlra_quantize_rtn.restype = i32
        L.mlra_quantize_rtn.argtypes = [vp, i32, i64, i64, i32, i64, vp, vp, vp, vp]
        L.mlra_dp_unique_id.restype = i32
        L.mlra_dp_unique_id.argtypes = [vp]
        L.mlra_dp_init.restype = i32
        L.mlra_dp_init.argtypes = [i32, i32, vp, C.POINTER(vp)]
        L.mlra_allreduce_lora_grads.restype = i32
        L.mlra_allreduce_lora_grads.argtypes = [vp, vp, u64, vp]
        L.mlra_dp_destroy.restype = None
        L.mlra_dp_destroy.argtypes = [vp]
        L.mlra_mix_seed.restype = u64
        L.mlra_mix_seed.argtypes = [u64, u64]
        L.mlra_gaussian_fill.restype = None
        L.mlra_gaussian_fill.argtypes = [u64, vp, u64, C.c_double, C.c_double]
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != MLRA_OK:
        msg = lib().mlra_last_error().decode()
        fk, off = None, 0
        if status == 7:
            o = C.c_uint64()
            k = lib().mlra_last_format_error(C.byref(o))
            if k >= 0:
                fk, off = FORMAT_KINDS.get(k), o.value
        raise MlraError(status, msg, fk, off)
