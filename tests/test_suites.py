"""Run-record schema and bench suites (metrics.py:15-119, bench.py:79-145 of
the reference) against CSV written by the reference's own suites
(tests/golden/suites_*.csv, make_golden.py).  Time-valued cells (wall,
speedup, busy, idle) are measurements and are compared for shape only;
dynamic-mode per-worker cells depend on the reference's thread schedule,
so those rows are compared on the run-level columns and the total."""

import csv
import io
import os

import pytest

from paper_1406_5687_b200 import metrics as M
from paper_1406_5687_b200.results import RankMetrics, RunResult

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TIME_COLS = {"wall_time", "speedup", "busy_time", "idle_time"}
SCHEDULE_COLS = {"triangles", "data_msgs_sent", "bytes_sent", "requests_sent", "tasks_executed"}


def _rows(text):
    return list(csv.DictReader(io.StringIO(text)))


def test_run_record_formatting_cpu():
    """Header, per-rank rows, det integer times, error rows (CPU only)."""
    m0 = RankMetrics(rank=0, nranks=2, triangles=5, data_msgs_sent=1, bytes_sent=24, busy_time=3.0,
                     partition_bytes=40)
    m1 = RankMetrics(rank=1, nranks=2, triangles=7, idle_time=2.0)
    rec = M.RunRecord.from_result("space-surrogate", 2, "predsum", "g", 0, "det", 12,
                                  RunResult(results=[12, None], metrics=[m0, m1], wall=9.0))
    err = M.RunRecord(algo="dynamic", ranks=1, cost="degree", graph="g", seed=1, backend="par", wall_time=0.0,
                      total=0, status="error", error="boom")
    buf = io.StringIO()
    M.write_run_csv([rec, err], buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == ",".join(M.RUN_COLUMNS)
    assert lines[1] == "count,space-surrogate,normal,2,predsum,g,0,det,ok,9,,0,5,1,24,0,0,3,0,40"
    assert lines[2] == "count,space-surrogate,normal,2,predsum,g,0,det,ok,9,,1,7,0,0,0,0,0,2,0"
    assert lines[3] == "count,dynamic,normal,1,degree,g,1,par,error:boom,0.000000,,,,,,,,,,"
    mem = io.StringIO()
    M.write_memory_csv([{"graph": "g", "d": 4, "ranks": 2, "cost": "predsum", "bytes_nonoverlap_max": 8,
                         "bytes_overlap_max": 16, "ratio": "2.0000"}], mem)
    assert mem.getvalue() == ",".join(M.MEMORY_COLUMNS) + "\ng,4,2,predsum,8,16,2.0000\n"


def test_golden_csv_schema_cpu():
    ref = open(os.path.join(HERE, "suites_run.csv")).read()
    assert ref.splitlines()[0].split(",") == M.RUN_COLUMNS
    mem = open(os.path.join(HERE, "suites_memory.csv")).read()
    assert mem.splitlines()[0].split(",") == M.MEMORY_COLUMNS


@pytest.mark.gpu
def test_suites_match_reference_csv():
    from paper_1406_5687_b200 import CostKind
    from paper_1406_5687_b200 import suites as S

    g = S.pa_graph(2000, 10, 3)
    label = S.pa_label(2000, 10, 3)
    pred, deg = CostKind.PRED_SUM, CostKind.DEGREE
    recs = S.bench_strong(g, label, "space-surrogate", [2, 4], pred, "par", 0)
    recs += S.bench_strong(g, label, "space-direct", [2, 3], pred, "par", 0)
    recs += S.bench_weak(400, 8, "space-surrogate", [1, 2, 3], pred, "par", 1)
    recs += S.bench_idle(g, label, 4, deg, 2, "par", 5)
    recs.append(S._record("space-surrogate", g, label, 0, pred, "par", 0, "count"))
    buf = io.StringIO()
    M.write_run_csv(recs, buf)
    got = _rows(buf.getvalue())
    ref = _rows(open(os.path.join(HERE, "suites_run.csv")).read())
    assert len(got) == len(ref)
    totals_got, totals_ref = {}, {}
    for a, b in zip(got, ref):
        dyn = a["algo"] == "dynamic" and a["mode"] == "normal"
        for col in M.RUN_COLUMNS:
            if col in TIME_COLS:
                assert (a[col] == "") == (b[col] == ""), col
            elif dyn and col in SCHEDULE_COLS:
                continue
            else:
                assert a[col] == b[col], (col, a, b)
        key = (a["suite"], a["algo"], a["mode"], a["ranks"], a["seed"], a["graph"])
        if a["triangles"]:
            totals_got[key] = totals_got.get(key, 0) + int(a["triangles"])
            totals_ref[key] = totals_ref.get(key, 0) + int(b["triangles"])
    assert totals_got == totals_ref

    mem = io.StringIO()
    M.write_memory_csv(S.bench_memory(1500, [4, 8, 12], 4, pred, 2), mem)
    assert mem.getvalue() == open(os.path.join(HERE, "suites_memory.csv")).read()
