"""Run records, aggregation and JSONL in the reference's format
(src/bench.cpp:34-330): CPU tests on hand-built records, a GPU test that
runs real solves through run_single."""
import json

import pytest

from paper_2406_00809_b200 import runrecord as rr


def rec(mid, pc, status, iauc=None, tauc=None, final=None):
    r = {"matrix_id": mid, "precond": pc, "status": status, "history": [(0, 1.0, 0.0)],
         "construct_secs": 0.5, "solve_secs": 1.5}
    if iauc is not None:
        r.update(iter_auc=iauc, time_auc=tauc, final_relres=final)
    return r


def test_percentiles_nearest_rank_lower():
    assert rr._percentiles_lower([]) == []
    assert rr._percentiles_lower([4.0, 1.0, 3.0, 2.0]) == [1.0, 2.0, 3.0, 4.0]
    assert rr._percentiles_lower([5.0]) == [5.0] * 4
    assert rr._percentiles_lower([3.0, 1.0, 2.0]) == [1.0, 2.0, 3.0, 3.0]


def test_aggregate_counts_failures_and_margins():
    recs = [
        rec("m1", "none", "maxiters", 10.0, 5.0, 1e-2),
        rec("m1", "gnp", "converged", 4.0, 6.0, 1e-8),
        rec("m1", "jacobi", "maxiters", 8.0, 2.0, 1e-4),
        rec("m2", "none", "converged", 3.0, 1.0, 1e-9),
        rec("m2", "gnp", "construction_failure"),
        rec("m3", "gnp", "solution_failure"),
    ]
    a = rr.aggregate(recs)
    assert a["best_by_iter_auc"] == {"gnp": 1, "none": 1}
    assert a["best_by_time_auc"] == {"jacobi": 1, "none": 1}
    assert a["failures"] == {"gnp": {"construction_failure": 1, "solution_failure": 1}}
    assert a["matrices_with_success"] == 2
    # gnp best by iter on m1; runner-up by iter_auc is jacobi: 1e-4 / 1e-8
    assert a["gnp_margin_by_iter"] == [pytest.approx(1e4)] * 4
    assert a["gnp_margin_by_time"] == []
    j = json.loads(rr.aggregate_to_json(a))
    assert j["margin_percentiles"] == [25, 50, 75, 100]


def test_record_json_roundtrip(tmp_path):
    recs = [rec("a", "gnp", "converged", 1.25, 0.5, 3e-9), rec("b", "ilu0", "construction_failure")]
    line = rr.record_to_json(recs[0])
    assert line.startswith('{"construct_secs":0.5,"final_relres":3e-09,"history":[[0,1.0,0.0]]')
    assert "iter_auc" not in rr.record_to_json(recs[1])
    p = tmp_path / "runs.jsonl"
    rr.write_records_jsonl(str(p), recs)
    back = rr.read_records_jsonl(str(p))
    assert back[0] == recs[0]
    assert back[1]["status"] == "construction_failure" and "iter_auc" not in back[1]


@pytest.mark.gpu
def test_run_single_gpu(gnp, cuda):
    a = gnp.prescale(gnp.gen_convection_diffusion(16, 0.5), 8.0)
    p, _ = gnp.train(a, steps=5, batch=8, spectral=4, arnoldi_m=10, d=4, hidden=8, layers=2)
    recs = [rr.run_single(a, "cd16", pc, params=p if pc == "gnp" else None, rtol=1e-6, maxiters=40,
                          restart=10) for pc in ("none", "jacobi", "gnp", "ilu0")]
    for r in recs[:3]:
        assert r["status"] in ("converged", "maxiters")
        assert r["history"][0][0] == 0 and r["iter_auc"] == gnp.iter_auc(r["history"], 1e-6)
        assert r["final_relres"] == r["history"][-1][1]
    assert recs[3]["status"] == "construction_failure"
    t = rr.run_single(a, "cd16", "none", rtol=1e-12, stop_mode="timeout", timeout_budget=0.05)
    assert t["status"] in ("timeout", "converged")
    a2 = rr.aggregate(recs)
    assert a2["matrices_with_success"] == 1
    assert rr.record_from_json(rr.record_to_json(recs[2]))["status"] == recs[2]["status"]
