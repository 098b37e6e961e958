"""Host-side selection sets (no torch): what the GPU path hands back to a caller of the
reference's API.

Contract (pkg/src/layerreuse/attention.py): `TopKSet` (:108-140) is a token selection of at
most `budget` distinct ascending indices; `BlockSet` (:143-182) a selection of distinct
ascending block ids of width `block_size`. Construction canonicalises to tuples of Python
ints and raises the reference's exception types (InvalidInputError for a bad budget or
width, InvalidSelectionError for a bad index list).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InvalidInputError, InvalidSelectionError

__all__ = ["TopKSet", "BlockSet"]


def _ascending_ids(values, noun: str, empty: str) -> tuple:
    """`values` as a tuple of ints, non-empty, non-negative and strictly increasing; `noun`
    names the entries in the error text, `empty` is the message for no entries."""
    ids = tuple(map(int, values))
    if len(ids) == 0:
        raise InvalidSelectionError(empty)
    arr = np.asarray(ids, dtype=np.int64)
    if int(arr.min()) < 0:
        raise InvalidSelectionError(f"{noun} indices must be non-negative")
    if arr.size > 1 and not bool(np.all(arr[1:] > arr[:-1])):
        raise InvalidSelectionError(f"{noun} indices must be strictly ascending")
    return ids


def _positive(value: int, name: str) -> None:
    if value < 1:
        raise InvalidInputError(f"{name} must be >= 1, got {value}")


@dataclass(frozen=True)
class TopKSet:
    """A token selection: distinct ascending indices, at most `budget` of them."""

    indices: tuple
    budget: int

    def __post_init__(self) -> None:
        _positive(self.budget, "budget")
        ids = _ascending_ids(self.indices, "token",
                             "selection must contain at least one index")
        if len(ids) > self.budget:
            raise InvalidSelectionError(
                f"selection holds {len(ids)} indices but budget is {self.budget}")
        object.__setattr__(self, "indices", ids)

    @property
    def size(self) -> int:
        return len(self.indices)


@dataclass(frozen=True)
class BlockSet:
    """A block selection: distinct ascending block ids of `block_size` tokens each; the
    token coverage of a cache of n tokens truncates the final block at n."""

    block_indices: tuple
    block_size: int

    def __post_init__(self) -> None:
        _positive(self.block_size, "block_size")
        object.__setattr__(self, "block_indices",
                           _ascending_ids(self.block_indices, "block",
                                          "block selection must contain at least one block"))

    @property
    def size(self) -> int:
        return len(self.block_indices)

    def token_coverage(self, n: int):
        if n < 1:
            raise InvalidInputError(f"cache length must be >= 1, got {n}")
        starts = np.asarray(self.block_indices, dtype=np.int64) * self.block_size
        beyond = np.nonzero(starts >= n)[0]
        if beyond.size:
            j = int(beyond[0])
            raise InvalidSelectionError(
                f"block {self.block_indices[j]} starts at token {int(starts[j])}, "
                f"beyond cache length {n}")
        ends = np.minimum(starts + self.block_size, n)
        return np.concatenate([np.arange(s, e, dtype=np.int64) for s, e in zip(starts, ends)])
