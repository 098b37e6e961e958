"""Host-side layer policy: FULL/REUSE actions and the lexicographic DP planner.

Mirrors the reference's planning interface (pkg/src/layerreuse/policy.py): `Action`
(:39-41), `LayerPolicy` (:58-116), `dp_optimize` (:143-208) with its tie rule (:211-223),
`validate_policy` (:273-307) and `static_jump_policy` (:310-336). The DP is O(L^2) host
work (north_star: "the DP policy search stays host-side"); its output must be
bit-identical to the reference on the same matrix, so the objective, the inclusive
threshold and the credit accumulation order are kept exactly.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass

from ._canon import FORMAT_VERSION, payload_hash
from .errors import InvalidInputError
from .profiling import SimilarityMatrix

__all__ = [
    "Action",
    "LayerPolicy",
    "dp_optimize",
    "brute_force_policy",
    "BRUTE_FORCE_MAX_LAYERS",
    "validate_policy",
    "static_jump_policy",
    "policy_from_actions",
]


class Action(enum.Enum):
    """Per-layer action (policy.py:39-41)."""

    FULL = "full"
    REUSE = "reuse"


@dataclass(frozen=True)
class LayerPolicy:
    """Actions plus the FULL layer each layer takes its selection from (policy.py:58-116).

    sources[j] == j exactly for FULL layers. Only structural shape is enforced here;
    semantic checks live in `validate_policy`.
    """

    actions: tuple
    sources: tuple
    theta: float | None
    full_count: int
    cum_similarity: float | None
    matrix_hash: str | None

    def __post_init__(self) -> None:
        actions = tuple(self.actions)
        sources = tuple(int(s) for s in self.sources)
        if not actions:
            raise InvalidInputError("a policy must cover at least one layer")
        if len(actions) != len(sources):
            raise InvalidInputError(f"{len(actions)} actions but {len(sources)} sources")
        if not all(isinstance(a, Action) for a in actions):
            raise InvalidInputError("actions must be Action values")
        if not all(0 <= s < len(actions) for s in sources):
            raise InvalidInputError("sources must be layer indices")
        if self.full_count != sum(a is Action.FULL for a in actions):
            raise InvalidInputError("full_count does not match the actions")
        object.__setattr__(self, "actions", actions)
        object.__setattr__(self, "sources", sources)

    @property
    def num_layers(self) -> int:
        return len(self.actions)

    def action_bytes(self) -> bytes:
        """The policy vector the C ABI takes (1 = FULL, 0 = REUSE)."""
        return bytes(1 if a is Action.FULL else 0 for a in self.actions)

    def canonical_payload(self) -> dict:
        return {
            "version": FORMAT_VERSION,
            "kind": "layer-policy",
            "L": self.num_layers,
            "theta": self.theta,
            "actions": [a.value for a in self.actions],
            "sources": [None if a is Action.FULL else s for a, s in zip(self.actions, self.sources)],
            "fullCount": self.full_count,
            "cumSimilarity": self.cum_similarity,
            "matrixHash": self.matrix_hash,
        }

    def sha256(self) -> str:
        return payload_hash(self.canonical_payload())


def _theta(theta) -> float:
    if not isinstance(theta, (int, float)) or not 0.0 <= float(theta) <= 1.0:
        raise InvalidInputError(f"theta must lie in [0, 1], got {theta}")
    return float(theta)


def policy_from_actions(actions) -> LayerPolicy:
    """Policy for an explicit action vector; a REUSE layer's source is the most recent
    FULL layer below it, which is what the engine actually reads (engine.py:173,185-194)."""
    acts = tuple(a if isinstance(a, Action) else Action(a) for a in actions)
    if not acts:
        raise InvalidInputError("a policy must cover at least one layer")
    sources, cur = [], 0
    for j, a in enumerate(acts):
        if a is Action.FULL:
            cur = j
        sources.append(cur)
    return LayerPolicy(acts, tuple(sources), None, sum(a is Action.FULL for a in acts), None, None)


def dp_optimize(matrix: SimilarityMatrix, theta: float) -> LayerPolicy:
    """Fewest FULL layers, then most similarity credit, for an inclusive threshold.

    State (i, j) = "layer j reuses FULL layer i" (i == j: layer j is FULL). The frontier
    at layer j holds, for every live source i, the best (full_count, credit, back)
    reaching it. Extending to j + 1: keep the chain if M[i][j+1] >= theta (credit
    += M[i][j+1]) or open a chain at j + 1 (full_count + 1, credit + 1). Candidates are
    offered in ascending source order and replace the incumbent only when strictly
    better, so exact ties keep the smaller source — the reference rule
    (policy.py:143-223), which makes the result bit-identical to exhaustive search.
    """
    theta = _theta(theta)
    L = matrix.num_layers
    M = matrix.values
    # frontier[i] = (full_count, credit, back) for layer j; history keeps the diagonal
    # cells, the only ones backtracking needs.
    frontier: dict[int, tuple[int, float, int]] = {0: (1, 1.0, -1)}
    opened: list[tuple[int, float, int]] = [(1, 1.0, -1)]
    for j in range(L - 1):
        nxt: dict[int, tuple[int, float, int]] = {}
        best_open: tuple[int, float, int] | None = None
        for i in sorted(frontier):
            fc, cr, _ = frontier[i]
            m = float(M[j + 1, i])
            if m >= theta:
                cand = (fc, cr + m, i)
                inc = nxt.get(i)
                if inc is None or _strictly_better(cand, inc):
                    nxt[i] = cand
            cand = (fc + 1, cr + 1.0, i)
            if best_open is None or _strictly_better(cand, best_open):
                best_open = cand
        nxt[j + 1] = best_open
        opened.append(best_open)
        frontier = nxt
    best_i, best = -1, None
    for i in sorted(frontier):
        if best is None or _strictly_better(frontier[i], best):
            best_i, best = i, frontier[i]
    sources = [0] * L
    i = best_i
    for j in range(L - 1, -1, -1):
        sources[j] = i
        if i == j and j > 0:
            i = opened[j][2]
    actions = tuple(Action.FULL if s == j else Action.REUSE for j, s in enumerate(sources))
    return LayerPolicy(actions, tuple(sources), theta, best[0], best[1], matrix.sha256())


# policy.py:36 — the exhaustive planner refuses larger stacks (2^(L-1) sequences)
BRUTE_FORCE_MAX_LAYERS = 14


def brute_force_policy(matrix: SimilarityMatrix, theta: float) -> LayerPolicy:
    """Exhaustive planner (policy.py:226-270), the reference's cross-check of dp_optimize
    (acceptance criterion 01, tests/test_acceptance.py:34-56).

    Every feasible action sequence is visited by a depth-first walk that extends a prefix
    one layer at a time (a REUSE step is taken only when it clears the inclusive
    threshold, so infeasible prefixes are cut at their first violation instead of being
    enumerated to the end). Credit is accumulated in ascending layer order along the walk,
    as the reference sums it, and sequences compare by (FULL count, -credit, sources read
    from the last layer down): the same objective and tie order as dp_optimize.
    """
    theta = _theta(theta)
    L = matrix.num_layers
    if L > BRUTE_FORCE_MAX_LAYERS:
        raise InvalidInputError(
            f"brute force is limited to {BRUTE_FORCE_MAX_LAYERS} layers, got {L}")
    M = matrix.values
    best = [None]  # (key, sources, fulls, credit)
    sources = [0] * L

    def walk(j: int, fulls: int, credit: float) -> None:
        if j == L:
            key = (fulls, -credit, tuple(reversed(sources)))
            if best[0] is None or key < best[0][0]:
                best[0] = (key, list(sources), fulls, credit)
            return
        # FULL at j
        sources[j] = j
        walk(j + 1, fulls + 1, credit + 1.0)
        # REUSE at j: inherit layer j-1's source if the overlap clears theta
        src = sources[j - 1]
        m = float(M[j, src])
        if m >= theta:
            sources[j] = src
            walk(j + 1, fulls, credit + m)

    sources[0] = 0
    walk(1, 1, 1.0)
    _, srcs, fulls, credit = best[0]
    actions = tuple(Action.FULL if s == j else Action.REUSE for j, s in enumerate(srcs))
    return LayerPolicy(actions, tuple(srcs), theta, fulls, credit, matrix.sha256())


def _strictly_better(a: tuple, b: tuple) -> bool:
    if a[0] != b[0]:
        return a[0] < b[0]
    return a[1] > b[1]


def validate_policy(policy: LayerPolicy, matrix: SimilarityMatrix, theta: float) -> list:
    """(layer, constraint) violations of a policy (policy.py:273-307)."""
    theta = _theta(theta)
    if policy.num_layers != matrix.num_layers:
        raise InvalidInputError(
            f"policy covers {policy.num_layers} layers, matrix {matrix.num_layers}"
        )
    out = []
    if policy.actions[0] is not Action.FULL:
        out.append((0, "first-layer-full"))
    for j, (a, s) in enumerate(zip(policy.actions, policy.sources)):
        if a is Action.FULL:
            if s != j:
                out.append((j, "self-source"))
            continue
        if j == 0:
            continue
        if s >= j or policy.actions[s] is not Action.FULL:
            out.append((j, "source-not-full"))
            continue
        if s != policy.sources[j - 1]:
            out.append((j, "chain"))
        if matrix.overlap(s, j) < theta:
            out.append((j, "threshold"))
    return out


def static_jump_policy(num_layers: int, stride: int) -> LayerPolicy:
    """FULL every `stride` layers, REUSE in between (policy.py:310-336)."""
    if num_layers < 1:
        raise InvalidInputError(f"num_layers must be >= 1, got {num_layers}")
    if stride < 1:
        raise InvalidInputError(f"stride must be >= 1, got {stride}")
    acts = tuple(Action.FULL if j % stride == 0 else Action.REUSE for j in range(num_layers))
    srcs = tuple((j // stride) * stride for j in range(num_layers))
    return LayerPolicy(acts, srcs, None, sum(a is Action.FULL for a in acts), None, None)
