"""NL2SQL workflow semantics for the wall-clock pool runtime.

The per-workflow outcomes must be bit-exact with the reference (north star), and
the reference makes them timing-independent: every draw is a pure function of
(seed, label, index) (stagesim/rng.py:26-29). This module restates exactly the
pieces the runtime needs, for the shipped NL2SQL workflow
(stagesim/workloads.py:82-120):

  * stream_uniform            — stagesim/rng.py:26-29
  * uniform sample / sample_int — stagesim/dists.py:76-92
  * outcome pick (cumulative, last positive-mass outcome absorbs rounding)
                              — stagesim/simulation.py:584-594
  * next_step with the retry budget on the executor->fixer loop edge
                              — stagesim/workflow.py:320-339 (the loop header is
                                the executor: it is entered from the generator,
                                workflow.py:241-274)
  * per-stage draw labels     — stagesim/simulation.py:526-527 (prompt/output),
                                :606 (outcome), :687 (tool service time)

tests/test_workflow_host.py pins it against the reference's own traces.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

GENERATOR = "sql_generator"
EXECUTOR = "sql_executor"
FIXER = "sql_fixer"
SUCCESS = "Success"
FAILURE = "Failure"

_U64 = 2 ** 64


def stream_uniform(seed: int, label: str, index: int) -> float:
    digest = hashlib.sha256(f"{seed}|{label}|{index}".encode()).digest()
    return (int.from_bytes(digest[:8], "big") + 1) / _U64


@dataclass(frozen=True)
class Uniform:
    low: float
    high: float

    def sample(self, u: float) -> float:
        return self.low + u * (self.high - self.low)

    def sample_int(self, u: float) -> int:
        lo, hi = int(self.low), int(self.high)
        return min(hi, lo + int(u * (hi - lo + 1)))

    def mean(self) -> float:
        return 0.5 * (self.low + self.high)


@dataclass(frozen=True)
class Constant:
    value: float

    def sample(self, u: float) -> float:
        return self.value

    def sample_int(self, u: float) -> int:
        return int(round(self.value))

    def mean(self) -> float:
        return self.value


@dataclass(frozen=True)
class Nl2Sql:
    """The workflow's knobs (stagesim/workloads.py:57-78 defaults, budget per config)."""

    p_fail: float = 0.5
    p_syntax_err: float = 0.25
    p_empty_result: float = 0.25
    retry_budget: int = 5
    slo_seconds: float = 30.0
    generator_prefix_tokens: int = 1000
    fixer_prefix_tokens: int = 1000
    prompt_tokens: object = field(default_factory=lambda: Uniform(100, 300))
    output_tokens: object = field(default_factory=lambda: Uniform(50, 150))
    executor_service_time: object = field(default_factory=lambda: Uniform(0.1, 0.4))

    def outcomes(self, stage: str) -> list[tuple[str, float, str]]:
        if stage == GENERATOR:
            return [("generated", 1.0, EXECUTOR)]
        if stage == FIXER:
            return [("fixed", 1.0, EXECUTOR)]
        return [("success", 1.0 - self.p_fail, SUCCESS),
                ("syntax_err", self.p_syntax_err, FIXER),
                ("empty_result", self.p_empty_result, FIXER)]

    def prefix(self, stage: str) -> int:
        return self.generator_prefix_tokens if stage == GENERATOR else self.fixer_prefix_tokens


def pick_outcome(outcomes, u: float) -> tuple[str, str]:
    cum = 0.0
    chosen = None
    for label, prob, target in outcomes:
        if prob <= 0.0:
            continue
        chosen = (label, target)
        cum += prob
        if u <= cum:
            break
    return chosen


class Workflow:
    """One request's walk through generator -> executor -> {done | fixer -> executor ...}."""

    __slots__ = ("rid", "spec", "seed", "stage", "retries", "visits", "history", "terminal",
                 "arrival", "done_time")

    def __init__(self, rid: int, spec: Nl2Sql, seed: int, arrival: float = 0.0) -> None:
        self.rid = rid
        self.spec = spec
        self.seed = seed
        self.stage = GENERATOR
        self.retries = 0
        self.visits: dict[str, int] = {}
        self.history: list[tuple[str, str]] = []
        self.terminal: str | None = None
        self.arrival = arrival
        self.done_time: float | None = None

    def _draw(self, kind: str, stage: str) -> float:
        label = f"req:{self.rid}:{kind}:{stage}"
        return stream_uniform(self.seed, label, self.visits[stage] - 1)

    def enter(self) -> tuple[int, int] | float:
        """Enter the current stage: (prompt, output) tokens for an LLM stage, or the
        tool service time for the executor (stagesim/simulation.py:521-534, :684-690)."""
        self.visits[self.stage] = self.visits.get(self.stage, 0) + 1
        if self.stage == EXECUTOR:
            return self.spec.executor_service_time.sample(self._draw("tool", EXECUTOR))
        p = self.spec.prompt_tokens.sample_int(self._draw("prompt", self.stage))
        o = self.spec.output_tokens.sample_int(self._draw("output", self.stage))
        return p, o

    def finish(self) -> str | None:
        """Apply the current stage's outcome; returns the next stage or None when done."""
        outs = self.spec.outcomes(self.stage)
        if len(outs) == 1:
            label, target = outs[0][0], outs[0][2]
        else:
            label, target = pick_outcome(outs, self._draw("outcome", self.stage))
        self.history.append((self.stage, label))
        if target in (SUCCESS, FAILURE):
            self.terminal = target
            return None
        if self.stage == EXECUTOR and target == FIXER:  # the budgeted loop edge
            if self.retries >= self.spec.retry_budget:
                self.terminal = FAILURE
                return None
            self.retries += 1
        self.stage = target
        return target
