"""Host mapping of the device flag words (include/hylra.h enum hylra_flag) onto the
reference's exceptions: out-of-range index -> InvalidSelectionError (attention.py:256-259),
non-finite scores or cache -> NumericInputError (attention.py:43-44), and the float64
refinement being skipped -> SelectionPrecisionWarning, or InvalidSelectionError when strict."""
import warnings

import pytest

from paper_2602_00777_b200 import _abi
from paper_2602_00777_b200.errors import (CudaError, InvalidSelectionError, NumericInputError,
                                          SelectionPrecisionWarning)


def test_clear_words_pass():
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        _abi.raise_for_flags([0, 0])
        _abi.raise_for_flags([0, 0], strict=True)


@pytest.mark.parametrize("bit,exc", [(_abi.FLAG_INDEX_OUT_OF_RANGE, InvalidSelectionError),
                                     (_abi.FLAG_NON_FINITE_SCORE, NumericInputError),
                                     (_abi.FLAG_NON_FINITE_CACHE, NumericInputError),
                                     (_abi.FLAG_INTERNAL, CudaError)])
def test_error_bits_raise(bit, exc):
    with pytest.raises(exc):
        _abi.raise_for_flags([bit, 0])
    # an error bit wins over the precision warning
    with pytest.raises(exc):
        _abi.raise_for_flags([bit | _abi.FLAG_REFINE_SKIPPED, 3])


def test_refine_skipped_warns_with_row_count_or_raises_when_strict():
    with pytest.warns(SelectionPrecisionWarning, match="3 selection row"):
        _abi.raise_for_flags([_abi.FLAG_REFINE_SKIPPED, 3])
    with pytest.raises(InvalidSelectionError, match="float64"):
        _abi.raise_for_flags([_abi.FLAG_REFINE_SKIPPED, 1], strict=True)
