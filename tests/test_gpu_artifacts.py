"""GPU producers of the interop artifacts vs the reference's own (tests/golden/artifacts/):
run_full_trace with block sets (synthetic.py:237-301) and sensitivity_profile
(profiling.py:204-284), then written with formats.py and read back."""
from pathlib import Path

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

torch = pytest.importorskip("torch")

from paper_2602_00777_b200 import formats as fm  # noqa: E402
from paper_2602_00777_b200.engine import (build_similarity_matrix, hybrid_decode,  # noqa: E402
                                          run_full_trace)
from paper_2602_00777_b200.policy import dp_optimize  # noqa: E402
from paper_2602_00777_b200.profiling import sensitivity_profile  # noqa: E402
from paper_2602_00777_b200.results import fidelity_report  # noqa: E402
from refmodel import FixtureModel, load_npz  # noqa: E402

ART = Path(__file__).resolve().parent / "golden" / "artifacts"


@pytest.fixture(scope="module")
def model(golden_dir):
    z = load_npz(golden_dir / "artifacts_reference.npz")
    return FixtureModel(z["keys"], z["values"], z["queries"], int(z["context_len"]),
                        probe=z["probe"], rho=float(z["rho"]), probe_step=int(z["sens_step"]))


def test_trace_with_blocks_matches_reference(model, tmp_path):
    ref = fm.read_trace(str(ART / "trace.json"))
    tr = run_full_trace(model, 3, 12, block_size=4)
    for t in range(3):
        for l in range(6):
            assert tr.topk[t][l].indices == ref.topk[t][l].indices
            assert tr.blocks[t][l].block_indices == ref.blocks[t][l].block_indices
    rel = np.linalg.norm(tr.outputs - ref.outputs) / np.linalg.norm(ref.outputs)
    assert rel < 1e-5
    # the GPU trace's matrix and DP policy are the reference's, byte for byte
    m = build_similarity_matrix(tr)
    fm.write_similarity_matrix(m, str(tmp_path / "matrix.json"))
    assert (tmp_path / "matrix.json").read_bytes() == (ART / "matrix.json").read_bytes()
    pol = dp_optimize(m, 0.6)
    fm.write_policy(pol, str(tmp_path / "policy.json"))
    assert (tmp_path / "policy.json").read_bytes() == (ART / "policy.json").read_bytes()
    # a written GPU trace reads back with identical selections
    fm.write_trace(tr, str(tmp_path / "trace.json"))
    back = fm.read_trace(str(tmp_path / "trace.json"))
    assert back.topk == tr.topk and back.blocks == tr.blocks


def test_fidelity_report_of_gpu_run(model):
    ref = fm.read_trace(str(ART / "trace.json"))
    pol = fm.read_policy(str(ART / "policy.json"))
    run = hybrid_decode(model, pol, 12, 3)
    rep = fidelity_report(ref, run)
    doc = fm.read_run_result(str(ART / "run.json"))
    np.testing.assert_allclose(rep.rnmse.per_layer,
                               [0.0 if x is None else x for x in doc["fidelity"]["perLayerRnmse"]],
                               rtol=1e-4, atol=1e-6)  # FULL layers: fp32 vs float64 outputs
    full = [l for l, a in enumerate(pol.actions) if a.value == "full"]
    assert np.all(rep.selection_overlap[:, full] == 1.0)


def test_sensitivity_profile_matches_reference(model):
    ref = fm.read_sensitivity_report(str(ART / "sensitivity.json"))
    got = sensitivity_profile(model, ref.step, ref.budget)
    assert got.step == ref.step and got.budget == ref.budget
    np.testing.assert_allclose(got.rnmse, ref.rnmse, rtol=1e-4, atol=1e-7)
    np.testing.assert_allclose(got.kl, ref.kl, rtol=1e-4, atol=1e-7)
    # a budget covering the cache saturates the selection: both measures vanish
    sat = sensitivity_profile(model, ref.step, 10_000)
    assert np.all(np.abs(sat.rnmse) < 1e-6) and np.all(np.abs(sat.kl) < 1e-6)
