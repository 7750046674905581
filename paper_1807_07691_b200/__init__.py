"""B200-native gSMat (arXiv 1807.07691) SM-based join executor.

Drop-in for the reference package's load/index/query path
(/root/reference/pkg/src/gsmat/__init__.py:5-29): ``load`` puts the
predicate-partitioned store in HBM, ``execute(..., mode="gpu")`` runs a plan
as a chain of sm_100a CUDA kernels and returns a ``BindingTable``.
"""

from .errors import (
    DeviceMemoryError,
    GsmatError,
    ParseError,
    ResourceLimitError,
    StoreFormatError,
    UnknownIdError,
    UnknownPredicateError,
    UnsupportedFeatureError,
)
from .executor import (
    DEFAULT_ROW_BUDGET,
    BindingTable,
    ExecutionReport,
    ResultSummary,
    StepReport,
    execute,
    execute_batch,
    execute_summary,
    fingerprint_rows,
)
from .frontend import Plan, QueryGraph, TriplePattern, bind_constants, make_plan, parse_query
from .decode import decode_rows, format_term, result_tsv, write_tsv
from .ingest import build, parse_ntriples
from .storage import (DeviceStore, EncodedTriple, PredicateMatrix, StatEntry, Store, build_store, from_store,
                      load, persist)

__all__ = [
    "EncodedTriple",
    "PredicateMatrix",
    "Store",
    "build_store",
    "persist",
    "build",
    "parse_ntriples",
    "decode_rows",
    "format_term",
    "result_tsv",
    "write_tsv",
    "BindingTable",
    "DEFAULT_ROW_BUDGET",
    "DeviceStore",
    "ExecutionReport",
    "GsmatError",
    "DeviceMemoryError",
    "ParseError",
    "Plan",
    "QueryGraph",
    "ResourceLimitError",
    "StatEntry",
    "StepReport",
    "StoreFormatError",
    "TriplePattern",
    "UnknownIdError",
    "UnknownPredicateError",
    "UnsupportedFeatureError",
    "bind_constants",
    "execute",
    "execute_batch",
    "execute_summary",
    "fingerprint_rows",
    "ResultSummary",
    "from_store",
    "load",
    "make_plan",
    "parse_query",
]

__version__ = "0.1.0"
