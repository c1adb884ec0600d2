"""The experiment harness (paper_1402_6601_b200/cli.py): the reference's CLI
suite runs against it in tests/test_reference_suite.py; these cover the B200
extensions (--p2p, --execute) and planner parity of its rows."""
import csv
import io
import math

import pytest

import paper_1402_6601_b200 as H
from paper_1402_6601_b200.cli import CSV_COLUMNS, EXEC_COLUMNS, main


def _rows(capsys, *argv):
    assert main(list(argv)) == 0
    rows = list(csv.reader(io.StringIO(capsys.readouterr().out)))
    return rows[0], rows[1:]


def test_p2p_rows_match_the_planner(capsys):
    hdr, rows = _rows(capsys, "run", "--kernel", "cholesky", "--nt", "8", "--tile", "512", "--cpus", "4",
                      "--gpus", "4", "--switches", "4", "--bandwidth", "7.7e11", "--latency", "3e-6",
                      "--p2p", "1", "--scheduler", "dada", "--cp", "1")
    assert hdr == CSV_COLUMNS
    g = H.gen_cholesky(8, 512)
    plat = H.build_platform(4, 4, 4, 7.7e11, 3e-6, None, p2p=True)
    plan = H.make_plan(g, plat, H.make_scheduler("dada", alpha=0.5, cp=True), H.PerfModel(H.default_timing_table(512, 128)))
    r = rows[0]
    assert int(r[CSV_COLUMNS.index("bytes_d2d")]) == plan.bytes_d2d > 0
    assert int(r[CSV_COLUMNS.index("bytes_d2h")]) == 0
    assert float(r[CSV_COLUMNS.index("makespan_s")]) == plan.makespan


def test_ini_p2p_and_execute_needs_gpu_only_platform(tmp_path, capsys):
    cfg = tmp_path / "b200.ini"
    cfg.write_text("[platform]\ncpus = 4\ngpus = 2\nswitches = 2\np2p = 1\n[kernel]\nfamily = lu\nnt = 2\n")
    assert main(["validate", "--config", str(cfg)]) == 0
    assert main(["run", "--config", str(cfg), "--execute"]) == 2  # 2 CPU workers: no CPU fallback
    assert "error:" in capsys.readouterr().err


@pytest.mark.gpu
def test_execute_on_b200(capsys):
    hdr, rows = _rows(capsys, "run", "--kernel", "cholesky", "--nt", "8", "--tile", "512", "--cpus", "1",
                      "--gpus", "1", "--switches", "1", "--p2p", "1", "--scheduler", "dada", "--cp", "1",
                      "--execute")
    assert hdr == EXEC_COLUMNS
    r = rows[0]
    assert int(r[EXEC_COLUMNS.index("exec_bytes_h2d")]) == int(r[EXEC_COLUMNS.index("bytes_h2d")])
    assert float(r[EXEC_COLUMNS.index("residual")]) < 1e-14
    assert float(r[EXEC_COLUMNS.index("measured_gflops")]) > 0
