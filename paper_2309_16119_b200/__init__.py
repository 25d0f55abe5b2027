"""B200-native ModuLoRA linear layer (arXiv 2309.16119): fused dequant +
tcgen05 GEMM kernels for sm_100a behind the reference's hot-path API.

The compute lives in libmlra.so (include/mlra.h); this package is the host-side
mirror of the reference interface (see modulora.py)."""
from ._lib import MlraError, build, lib  # noqa: F401
from .ledger import (  # noqa: F401
    LayerDims, LedgerEvent, LedgerReport, MemoryLedger, Phase, ledger_assert_single_materialization)
from .modulora import (  # noqa: F401
    Cb2Matrix, Codebook2Quantizer, DeviceQuantizedMatrix, DoublingQuantizer, E8pMatrix,
    E8pQuantizer, IncoherentLayer, LoraAdapter, e8p_abs_table, e8p_decode, random_signs, rht,
    LpLinearContext, LpLinearFunction, LutMatrix, LutQuantizer, MaterializationStrategy, NF4_LEVELS, OptqQuantizer, ModuLoraLayer, ModuLoraLinearFunction, PackedCodes,
    QuantizedMatrix, QuantizerHook, RtnQuantizer, default_cb2_codebook, dequantize,
    dequantize_row, dequantize_tile, grads_of_adapter, init_adapter, layer_backward, layer_forward,
    lp_backward, lp_forward, make_layer, normal_float_levels, optq_workspace, pack_codes, quantized_matvec,
    quantized_matvec_transposed, unpack_codes, packed_word_count, parse_strategy, strategy_name)
