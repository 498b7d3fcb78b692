"""Evaluation records for GPU solves, in the reference's format.

Mirrors the run-record layer of the reference benchmark harness
(src/bench.cpp, include/gnp/bench.hpp) over this package's solver:

  run_single(...)          src/bench.cpp:53-116   one (matrix, preconditioner) solve,
                                                  b = A·1, construction + solve timed
  aggregate(records)       src/bench.cpp:223-263  best-by-AUC counts, failures, GNP margins
  record_to_json / record_from_json
                           src/bench.cpp:265-298  one JSON object per record
  write_records_jsonl / read_records_jsonl
                           src/bench.cpp:311-330
  aggregate_to_json        src/bench.cpp:300-309

Records are plain dicts with the reference's keys.  JSON text uses sorted keys
and compact separators, the layout nlohmann::json's dump() produces for these
objects.  Preconditioners this package does not serve ("gmres", "ilu0") end
as "construction_failure", like any construction error in the reference.
"""
from __future__ import annotations

import json
import math
import time

FAIL_OK = ("converged", "maxiters", "timeout", "breakdown_exact")


def _g():
    import paper_2406_00809_b200 as g

    return g


def run_single(matrix, matrix_id: str, precond: str, params=None, rtol: float = 1e-8,
               maxiters: int = 100, restart: int = 10, stop_mode: str = "maxiters",
               timeout_budget: float | None = None, timeout_secs: float | None = None,
               train_kwargs: dict | None = None) -> dict:
    """src/bench.cpp:53-116.  `matrix` is an already prescaled CsrMatrix;
    precond in none | jacobi | gmres | ilu0 | gnp ("gnp" trains with
    train_kwargs when params is None, inside the timed construction)."""
    g = _g()
    rec = {"matrix_id": matrix_id, "precond": precond, "status": "", "history": [],
           "construct_secs": 0.0, "solve_secs": 0.0}
    t0 = time.perf_counter()
    p = params
    try:
        if precond not in ("none", "jacobi", "gnp"):
            raise ValueError("preconditioner not served by this package: " + precond)
        if precond == "gnp" and p is None:
            p, _ = g.train(matrix, **(train_kwargs or {}))
    except Exception:
        rec["status"] = "construction_failure"
        rec["construct_secs"] = time.perf_counter() - t0
        return rec
    rec["construct_secs"] = time.perf_counter() - t0
    b = g.spmv(matrix, [1.0] * matrix.n)  # ground truth x = 1
    if stop_mode == "timeout":
        maxiters = 2 ** 31 - 1  # unbounded (the reference's SIZE_MAX/2; the device counter is int)
        timeout_secs = timeout_budget if timeout_budget is not None else (
            timeout_secs if timeout_secs is not None else 1.0)
    elif stop_mode != "maxiters":
        raise ValueError("stop_mode must be maxiters or timeout")
    t1 = time.perf_counter()
    try:
        out = g.solve(matrix, b, precond=precond, params=p if precond == "gnp" else None, rtol=rtol,
                      maxiters=maxiters, restart=restart, timeout_secs=timeout_secs)
        rec["solve_secs"] = time.perf_counter() - t1
        hist = [(int(i), float(r), float(t)) for i, r, t in out["history"]]
        rec["status"] = out["status"]
        rec["history"] = hist
        rec["iter_auc"] = g.iter_auc(hist, rtol)
        rec["time_auc"] = g.time_auc(hist, rtol)
        rec["final_relres"] = hist[-1][1]
    except Exception:
        rec["solve_secs"] = time.perf_counter() - t1
        rec["status"] = "solution_failure"
    return rec


def _percentiles_lower(values):
    """src/bench.cpp:211-221: 25/50/75/100 % by nearest-rank (lower)."""
    if not values:
        return []
    v = sorted(values)
    out = []
    for p in (0.25, 0.50, 0.75, 1.00):
        rank = int(math.ceil(p * len(v)))
        out.append(v[rank - 1 if rank > 0 else 0])
    return out


def aggregate(records) -> dict:
    """src/bench.cpp:223-263."""
    best_iter, best_time, failures = {}, {}, {}
    by_matrix = {}
    for r in records:
        by_matrix.setdefault(r["matrix_id"], []).append(r)
        if r["status"] not in FAIL_OK:
            failures.setdefault(r["precond"], {})
            failures[r["precond"]][r["status"]] = failures[r["precond"]].get(r["status"], 0) + 1
    margins_iter, margins_time = [], []
    with_success = 0
    for mid in sorted(by_matrix):
        ok = [r for r in by_matrix[mid] if r.get("iter_auc") is not None]
        if not ok:
            continue
        with_success += 1
        for key, counts, margins in (("iter_auc", best_iter, margins_iter),
                                     ("time_auc", best_time, margins_time)):
            best = ok[0]
            for r in ok:  # first strict minimum, in record order
                if r[key] < best[key]:
                    best = r
            counts[best["precond"]] = counts.get(best["precond"], 0) + 1
            if best["precond"] == "gnp" and len(ok) > 1 and best.get("final_relres") is not None:
                second = None
                for r in ok:
                    if r is best:
                        continue
                    if second is None or r[key] < second[key]:
                        second = r
                if (second is not None and second.get("final_relres") is not None
                        and best["final_relres"] > 0.0):
                    margins.append(second["final_relres"] / best["final_relres"])
    return {"best_by_iter_auc": best_iter, "best_by_time_auc": best_time, "failures": failures,
            "matrices_with_success": with_success,
            "gnp_margin_by_iter": _percentiles_lower(margins_iter),
            "gnp_margin_by_time": _percentiles_lower(margins_time)}


def record_to_json(r: dict) -> str:
    j = {k: r[k] for k in ("matrix_id", "precond", "status", "construct_secs", "solve_secs")}
    j["history"] = [[int(i), float(x), float(t)] for i, x, t in r["history"]]
    for k in ("iter_auc", "time_auc", "final_relres"):
        if r.get(k) is not None:
            j[k] = r[k]
    return json.dumps(j, sort_keys=True, separators=(",", ":"))


def record_from_json(line: str) -> dict:
    j = json.loads(line)
    r = {"matrix_id": j["matrix_id"], "precond": j["precond"], "status": j["status"],
         "history": [(int(e[0]), float(e[1]), float(e[2])) for e in j["history"]],
         "construct_secs": float(j["construct_secs"]), "solve_secs": float(j["solve_secs"])}
    for k in ("iter_auc", "time_auc", "final_relres"):
        if k in j:
            r[k] = float(j[k])
    return r


def aggregate_to_json(rep: dict) -> str:
    j = dict(rep)
    j["margin_percentiles"] = [25, 50, 75, 100]
    return json.dumps(j, sort_keys=True, indent=2)


def write_records_jsonl(path: str, records) -> None:
    with open(path, "w") as f:
        for r in records:
            f.write(record_to_json(r) + "\n")


def read_records_jsonl(path: str):
    with open(path) as f:
        return [record_from_json(line) for line in f if line.strip()]
