"""B200-native fp64 SpMV library (drop-in for the hot path of spmvkit,
the artifact of arXiv 1805.11938).

Public names mirror ``spmvkit``'s hot-path API (coo, formats, kernels,
features, select_format).  All compute runs in hand-written sm_100a CUDA
kernels in ``libspmvb.so`` (C ABI: include/spmvb.h) loaded with ctypes; the
package refuses to import if the library is missing (no CPU fallback).
"""

from . import _lib

_lib.load()  # fail loudly at import time if libspmvb.so is missing

from .coo import (  # noqa: E402
    INDEX_LIMIT,
    CooMatrix,
    MatrixMarketError,
    canonicalize,
    coo_equal,
    dense_spmv_oracle,
    read_matrix_market,
    row_nnz_histogram,
    write_matrix_market,
)
from .features import (  # noqa: E402
    FEATURE_NAMES,
    FeatureVector,
    ScalingParams,
    apply_scaling,
    extract_extra_features,
    extract_features,
    features_from_line,
    features_to_line,
    fit_scaling,
    read_features,
    write_features,
)
from .formats import (  # noqa: E402
    DEFAULT_MAX_GRID_CELLS,
    ConversionError,
    Csr5Matrix,
    CsrMatrix,
    EllMatrix,
    FormatMatrix,
    FormatTag,
    HybMatrix,
    SellMatrix,
    convert,
    hyb_typical_k,
    to_coo,
    to_csr,
    to_csr5,
    to_ell,
    to_hyb,
    to_sell,
)
from . import synth  # noqa: E402
from .harness import (  # noqa: E402
    BenchConfig,
    BenchRecord,
    bandwidth_estimate,
    bench_corpus,
    best_labels,
    discover_corpus,
    read_records,
    record_from_line,
    record_to_line,
    run_bench,
    spmv_bytes,
    spmv_flops,
    times_by_matrix,
    write_records,
)
from .kernels import (  # noqa: E402
    BoundCall, SpmvOperator, bind, bind_range, spmv, spmv_csr, spmv_csr5, spmv_csr5_push, spmv_csr5_tiles, spmv_ell, spmv_hyb, spmv_many, spmv_sell,
    spmv_sell_range,
)
from .relabel import DegreeOrder, RelabelledMatrix, power_iteration  # noqa: E402
from .model import (  # noqa: E402
    B200_SELECTOR_PARAMS,
    DecisionTreeModel,
    ModelIOError,
    default_model,
    load_model,
    predict,
    select_format,
    select_format_b200,
    select_format_measured,
)

__version__ = "0.1.0"
