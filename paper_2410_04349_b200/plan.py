"""The compiled execution path: the program the device interprets.

Format restated from the reference (pkg/src/ruleblock/planner/plan.py:218-300):
a flat instruction list of ``EvalPredicate(slot, fail_jump)`` and
``Checkpoint(rule_id)``; a true predicate falls through, a false one jumps
past its subtree; the first checkpoint reached names the witness rule.

The timing-based planner (cost MLP, selectivity sampling; plan.py:341-385)
stays out of scope.  ``plan_from_stats`` reproduces the deterministic part
of it -- cost-effectiveness ordering (plan.py:28-76), prefix-tree build
(plan.py:147-169), witness-probability scoring (plan.py:181-211) and DFS
compilation -- from caller-supplied cost / selectivity numbers, which is
how the reference's own tests freeze a plan (pkg/tests/conftest.py:41-47).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Mapping, Union

from .errors import ConfigError
from .rules import Predicate, predicate_universe


@dataclass(frozen=True)
class EvalPredicate:
    slot: int
    fail_jump: int


@dataclass(frozen=True)
class Checkpoint:
    rule_id: str


Instruction = Union[EvalPredicate, Checkpoint]


@dataclass
class ExecutionPath:
    instructions: list
    predicate_table: list
    rule_ids: list
    root_slots: list

    @property
    def n_slots(self) -> int:
        return len(self.predicate_table)

    def checkpoint_order(self) -> list[str]:
        return [i.rule_id for i in self.instructions if is_checkpoint(i)]


def is_checkpoint(ins) -> bool:
    """Duck-typed: works for the reference's instruction classes too."""
    return not hasattr(ins, "slot")


# ---------------------------------------------------------------------------
# Deterministic plan construction from given costs / selectivities


@dataclass
class _Node:
    edges: list = field(default_factory=list)  # [pred, child, cover(set), score]
    leaves: list = field(default_factory=list)


def plan_from_stats(rules, costs: Mapping[Predicate, float], sps: Mapping[Predicate, float]) -> ExecutionPath:
    universe = predicate_universe(rules)
    for p in universe:
        if p not in costs or p not in sps:
            raise ConfigError(f"cost/sp missing for {p.describe()}")
        if costs[p] <= 0:
            raise ConfigError(f"estimated cost must be positive, got {costs[p]}")
    # descending (1 - sp) / cost; ties: ascending cost, then first appearance
    keyed = sorted(
        range(len(universe)),
        key=lambda k: (-(1.0 - sps[universe[k]]) / costs[universe[k]], costs[universe[k]], k),
    )
    rank = {universe[k]: r for r, k in enumerate(keyed)}

    root = _Node()
    for rule in rules:
        node = root
        for p in sorted(rule.precondition, key=rank.__getitem__):
            edge = next((e for e in node.edges if e[0] == p), None)
            if edge is None:
                edge = [p, _Node(), set(), 0.0]
                node.edges.append(edge)
            edge[2].add(rule.rule_id)
            node = edge[1]
        node.leaves.append(rule.rule_id)

    wp = {}
    for rule in rules:
        w = 1.0
        for p in rule.precondition:
            w *= sps[p]
        wp[rule.rule_id] = w

    def score(node: _Node) -> None:
        for e in node.edges:
            e[3] = max(wp[r] for r in e[2])
            score(e[1])
        node.edges.sort(key=lambda e: -e[3])  # stable: insertion order on ties

    score(root)

    slots: dict = {}
    ins: list = []

    def emit(node: _Node) -> None:
        for rid in node.leaves:
            ins.append(Checkpoint(rid))
        for e in node.edges:
            s = slots.setdefault(e[0], len(slots))
            at = len(ins)
            ins.append(None)
            emit(e[1])
            ins[at] = EvalPredicate(s, len(ins))

    emit(root)
    table = sorted(slots, key=slots.__getitem__)
    return ExecutionPath(
        instructions=ins,
        predicate_table=table,
        rule_ids=[r.rule_id for r in rules],
        root_slots=[slots[e[0]] for e in root.edges],
    )


# ---------------------------------------------------------------------------
# Plain-data (JSON) form, used by the golden fixtures


def predicate_to_dict(p) -> dict:
    return {
        "lhs_attr": p.lhs_attr,
        "comparator": p.comparator,
        "rhs_attr": p.rhs_attr,
        "const": p.const,
        "measure": p.measure,
        "threshold": p.threshold,
    }


def path_to_dict(path) -> dict:
    return {
        "instructions": [
            ["C", i.rule_id] if is_checkpoint(i) else ["E", i.slot, i.fail_jump] for i in path.instructions
        ],
        "predicate_table": [predicate_to_dict(p) for p in path.predicate_table],
        "rule_ids": list(path.rule_ids),
        "root_slots": list(path.root_slots),
    }


def path_from_dict(d: dict) -> ExecutionPath:
    ins = [Checkpoint(x[1]) if x[0] == "C" else EvalPredicate(int(x[1]), int(x[2])) for x in d["instructions"]]
    return ExecutionPath(
        instructions=ins,
        predicate_table=[Predicate(**p) for p in d["predicate_table"]],
        rule_ids=list(d["rule_ids"]),
        root_slots=list(d["root_slots"]),
    )
