"""B200-native rule-evaluation engine for rule-based blocking.

Drop-in replacement of the hot path of the reference package ``ruleblock``
(HyperBlocker, arXiv 2410.04349): ``run_partition`` / ``run_cross`` evaluate
a compiled set of conjunctive blocking rules over every tuple pair of a
partition on one sm_100a GPU and return the surviving
``(t_tid, s_tid, rule_id)`` rows, bit-exact with the reference engine.
"""

from .encode import Encoded, RelationEncoding, compile_program
from .engine import (
    BlockStats,
    CandidateSet,
    EngineConfig,
    PairBitmaps,
    PathProgram,
    evaluate_pair,
    evaluate_pairs,
    RunStats,
    context,
    run_cross,
    run_crosses,
    run_partition,
    run_partitions,
    run_partition_rows,
    split_rows_by_pairs,
)
from .ingest import ColumnarRelation, load_relation
from .errors import ConfigError, DataParseError, RuleBlockError, RuleParseError, SchemaError, ValidationError
from .pipeline import BandingConfig, PipelineConfig, PipelineResult, iter_partitions, pipeline_run
from .plan import Checkpoint, EvalPredicate, ExecutionPath, plan_from_stats
from .scheduler import MultiDeviceEngine
from .relation import MISSING, DataPartition, Kind, Relation, Schema, TupleRecord, relation_from_rows
from .rules import MDRule, Predicate, RuleSet, parse_ruleset, predicate_universe

__version__ = "0.1.0"

__all__ = [
    "evaluate_pairs",
    "BandingConfig", "BlockStats", "ColumnarRelation", "load_relation", "CandidateSet", "MultiDeviceEngine", "PipelineConfig", "PipelineResult",
    "iter_partitions", "pipeline_run", "Checkpoint", "ConfigError", "DataParseError", "DataPartition", "Encoded",
    "EngineConfig", "PairBitmaps", "evaluate_pair", "EvalPredicate", "ExecutionPath", "Kind", "MDRule", "MISSING", "PathProgram", "Predicate",
    "Relation", "RelationEncoding", "RuleBlockError", "RuleParseError", "RuleSet", "RunStats", "Schema",
    "SchemaError", "TupleRecord", "ValidationError", "compile_program", "context", "parse_ruleset",
    "plan_from_stats", "predicate_universe", "relation_from_rows", "run_cross", "run_crosses", "run_partition", "run_partitions", "run_partition_rows", "split_rows_by_pairs",
]
