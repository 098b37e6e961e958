"""Artifact interop (reference formats.py / engine.py cost_model + fidelity_report): the
reference's own artifacts (tests/golden/artifacts/, written by the reference through
tests/golden/make_golden.py) load here, and re-writing them gives byte-identical files."""
import filecmp
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2602_00777_b200 import formats as fm
from paper_2602_00777_b200.errors import InvalidInputError
from paper_2602_00777_b200.policy import Action
from paper_2602_00777_b200.results import (DecodeRunResult, cost_model, fidelity_report,
                                           fidelity_tables)
from paper_2602_00777_b200.sets import BlockSet, TopKSet
from refmodel import load_npz

ART = Path(__file__).resolve().parent / "golden" / "artifacts"


@pytest.fixture(scope="module")
def z(golden_dir):
    return load_npz(golden_dir / "artifacts_reference.npz")


def _same_bytes(a, b):
    assert Path(a).read_bytes() == Path(b).read_bytes(), f"{a} != {b}"


def test_trace_roundtrip_bytes(tmp_path, z):
    tr = fm.read_trace(str(ART / "trace.json"))
    assert tr.budget == 12 and tr.block_size == 4 and tr.steps == 3
    assert tr.config.layers == 6 and tr.config.heads == 2
    np.testing.assert_array_equal(tr.queries, z["queries"])
    assert all(len(s.indices) == 12 for row in tr.topk for s in row)
    fm.write_trace(tr, str(tmp_path / "trace.json"))
    for name in ("trace.json", "trace.queries.bin", "trace.outputs.bin"):
        _same_bytes(ART / name, tmp_path / name)


def test_matrix_policy_sensitivity_roundtrip(tmp_path):
    m = fm.read_similarity_matrix(str(ART / "matrix.json"))
    fm.write_similarity_matrix(m, str(tmp_path / "m.json"))
    _same_bytes(ART / "matrix.json", tmp_path / "m.json")
    pol = fm.read_policy(str(ART / "policy.json"))
    assert pol.matrix_hash == m.sha256()
    fm.write_policy(pol, str(tmp_path / "p.json"))
    _same_bytes(ART / "policy.json", tmp_path / "p.json")
    rep = fm.read_sensitivity_report(str(ART / "sensitivity.json"))
    fm.write_sensitivity_report(rep, str(tmp_path / "s.json"))
    _same_bytes(ART / "sensitivity.json", tmp_path / "s.json")
    rows = fm.similarity_matrix_csv_rows(m)
    assert len(rows) == 21 and rows[0] == (0, 0, 1.0)


def test_cost_model_matches_reference(tmp_path):
    pol = fm.read_policy(str(ART / "policy.json"))
    fm.write_cost_report(cost_model(pol, 32768, 2048, head_dim=1024, bytes_per_elem=2),
                         str(tmp_path / "c.json"), contextLen=32768, budget=2048)
    _same_bytes(ART / "cost.json", tmp_path / "c.json")
    fm.write_cost_report(cost_model(pol, 1000, 7, block_size=128, head_dim=64),
                         str(tmp_path / "cb.json"))
    _same_bytes(ART / "cost_blocks.json", tmp_path / "cb.json")
    with pytest.raises(InvalidInputError):
        cost_model(pol, 0, 1)


def _run_from_fixture(z, pol, trace, block: bool):
    acts = pol.actions
    T, L = 3, len(acts)
    n0 = int(z["context_len"])
    sels, gathered = [], []
    for t in range(T):
        row_s, row_g, cur = [], [], None
        for l in range(L):
            if acts[l] is Action.FULL:
                cur = (BlockSet(tuple(z["runb_blocks"][t][l]), int(z["block_size"])) if block
                       else TopKSet(tuple(z["run_sets"][t][l]), int(z["budget"])))
                row_g.append(None)
            else:
                row_g.append(int(cur.token_coverage(n0 + t).shape[0]) if block else cur.size)
            row_s.append(cur)
        sels.append(tuple(row_s))
        gathered.append(tuple(row_g))
    outs = z["runb_outputs"] if block else z["run_outputs"]
    return DecodeRunResult(policy=pol, budget=3 if block else int(z["budget"]),
                           block_size=int(z["block_size"]) if block else 1, outputs=outs,
                           selections=tuple(sels),
                           fidelity=fidelity_tables(trace.outputs, outs),
                           full_score_computations=(pol.full_count,) * T, reuse_full_scans=0,
                           reuse_gathered_rows=tuple(gathered))


@pytest.mark.parametrize("block", [False, True])
def test_run_result_and_fidelity_report(tmp_path, z, block):
    pol = fm.read_policy(str(ART / "policy.json"))
    trace = fm.read_trace(str(ART / "trace.json"))
    run = _run_from_fixture(z, pol, trace, block)
    name = "run_blocks.json" if block else "run.json"
    fm.write_run_result(run, str(tmp_path / name))
    _same_bytes(ART / name, tmp_path / name)
    rep = fidelity_report(trace, run)
    pre = "fidb_" if block else "fid_"
    np.testing.assert_array_equal(rep.selection_overlap, z[pre + "overlap"])
    np.testing.assert_array_equal(rep.rnmse.per_step_layer, z[pre + "rnmse"])
    if not block:
        np.testing.assert_array_equal(rep.per_layer_overlap, z["fid_per_layer"])
        assert rep.rnmse.aggregate == float(z["fid_aggregate"])


def test_header_checks(tmp_path):
    bad = tmp_path / "x.json"
    bad.write_text('{"kind": "layer-policy", "version": "2.0"}')
    with pytest.raises(InvalidInputError):
        fm.read_policy(str(bad))
    with pytest.raises(InvalidInputError):
        fm.read_similarity_matrix(str(ART / "policy.json"))


@pytest.mark.skipif(not Path("/root/reference/pkg/src").exists(),
                    reason="the reference CLI exists only in the build container")
def test_reference_cli_reports_our_artifacts(tmp_path, z):
    """Artifacts written by this package feed the reference's `report` command."""
    pol = fm.read_policy(str(ART / "policy.json"))
    trace = fm.read_trace(str(ART / "trace.json"))
    fm.write_policy(pol, str(tmp_path / "policy.json"))
    fm.write_similarity_matrix(fm.read_similarity_matrix(str(ART / "matrix.json")),
                               str(tmp_path / "matrix.json"))
    fm.write_run_result(_run_from_fixture(z, pol, trace, False), str(tmp_path / "run.json"))
    out = tmp_path / "report"
    env = dict(os.environ, PYTHONPATH="/root/reference/pkg/src", PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run([sys.executable, "-m", "layerreuse", "report",
                        str(tmp_path / "policy.json"), str(tmp_path / "matrix.json"),
                        str(tmp_path / "run.json"), "--out", str(out)],
                       capture_output=True, text=True, env=env, cwd=tmp_path)
    assert r.returncode == 0, r.stderr
    assert (out / "policies.md").exists() and (out / "run.rnmse.csv").exists()
