"""B200-native exact KNN self-join engine (HybridKNN-Join hot path, arXiv 1810.04758).

The product is the C-ABI library ``libknnj_b200.so`` (include/knnj_c.h); this
package is its Python mirror of the reference ``knnjoin`` API.
"""
from ._capi import KnnjError, load_library  # noqa: F401
from .engine import (  # noqa: F401
    CandidateOutcome, Engine, KnnRunResult, ParameterSearchResult, RunConfig, derive_seed,
    ingest_dataset, parameter_search, read_binary_f64, read_text, run_hybrid, tsv_bytes, tsv_string, write_tsv,
)
from .synthetic import generate  # noqa: F401
