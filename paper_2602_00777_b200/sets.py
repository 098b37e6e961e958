"""Canonical selection sets (host-only; no torch).

Reference: pkg/src/layerreuse/attention.py — `TopKSet` (:108-140) and `BlockSet` (:143-182),
with the same canonical-form checks and error types.
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import InvalidInputError, InvalidSelectionError

__all__ = ["TopKSet", "BlockSet"]


@dataclass(frozen=True)
class TopKSet:
    """Canonical selection: distinct ascending indices plus the requested budget."""

    indices: tuple
    budget: int

    def __post_init__(self) -> None:
        ind = tuple(int(i) for i in self.indices)
        if self.budget < 1:
            raise InvalidInputError(f"budget must be >= 1, got {self.budget}")
        if not ind:
            raise InvalidSelectionError("selection must contain at least one index")
        if any(i < 0 for i in ind):
            raise InvalidSelectionError("token indices must be non-negative")
        if any(b <= a for a, b in zip(ind, ind[1:])):
            raise InvalidSelectionError("token indices must be strictly ascending")
        if len(ind) > self.budget:
            raise InvalidSelectionError(
                f"selection holds {len(ind)} indices but budget is {self.budget}")
        object.__setattr__(self, "indices", ind)

    @property
    def size(self) -> int:
        return len(self.indices)


@dataclass(frozen=True)
class BlockSet:
    """Canonical block selection (attention.py:143-182): distinct ascending block indices
    plus the block width; token_coverage(n) truncates the final block at n."""

    block_indices: tuple
    block_size: int

    def __post_init__(self) -> None:
        blocks = tuple(int(b) for b in self.block_indices)
        if self.block_size < 1:
            raise InvalidInputError(f"block_size must be >= 1, got {self.block_size}")
        if not blocks:
            raise InvalidSelectionError("block selection must contain at least one block")
        if any(b < 0 for b in blocks):
            raise InvalidSelectionError("block indices must be non-negative")
        if any(b2 <= b1 for b1, b2 in zip(blocks, blocks[1:])):
            raise InvalidSelectionError("block indices must be strictly ascending")
        object.__setattr__(self, "block_indices", blocks)

    @property
    def size(self) -> int:
        return len(self.block_indices)

    def token_coverage(self, n: int):
        import numpy as np
        if n < 1:
            raise InvalidInputError(f"cache length must be >= 1, got {n}")
        spans = []
        for b in self.block_indices:
            start = b * self.block_size
            if start >= n:
                raise InvalidSelectionError(
                    f"block {b} starts at token {start}, beyond cache length {n}")
            spans.append(np.arange(start, min(start + self.block_size, n), dtype=np.int64))
        return np.concatenate(spans)
