"""B200-native unified kernel-segregated stride-2 transpose convolution.

A drop-in for the segregated-engine path of the reference package `segconv`
(arXiv 2502.20493): same entry points, padding/output-size conventions and
error behaviour, with the arithmetic in hand-written sm_100a CUDA kernels
behind the C ABI of include/segb200.h.
"""

from .engines import (
    ENGINE_REFERENCE,
    ENGINE_SEGREGATED,
    ENGINES,
    ComparisonReport,
    EngineCounters,
    PreparedLayer,
    compare_outputs,
    layer_forward,
    prepare_layer,
    transpose_conv_reference,
    transpose_conv_reference_counted,
    transpose_conv_segregated,
    wait_host_copies,
    transpose_conv_segregated_counted,
)
from .errors import ShapeError, SpecError
from .segregation import SubKernelSet, merge_subkernels, segregate_kernel
from .stack import PreparedStack, prepare_stack
from . import tensor_io  # noqa: E402
from .spec import (
    EffectivePadding,
    TransposeConvSpec,
    effective_padding,
    memory_savings_bytes,
    mult_count_segregated,
    output_dims,
    subkernel_dims,
)

__all__ = [
    "ENGINE_REFERENCE", "ENGINE_SEGREGATED", "ENGINES", "ComparisonReport", "EffectivePadding", "EngineCounters",
    "PreparedLayer", "PreparedStack", "ShapeError", "SpecError", "SubKernelSet", "TransposeConvSpec",
    "compare_outputs", "effective_padding", "layer_forward", "memory_savings_bytes", "merge_subkernels",
    "mult_count_segregated", "output_dims", "prepare_layer", "prepare_stack", "segregate_kernel",
    "subkernel_dims", "transpose_conv_reference", "transpose_conv_reference_counted",
    "transpose_conv_segregated", "transpose_conv_segregated_counted",
    "wait_host_copies",
]
