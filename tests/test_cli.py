"""`rbe-cuda`, the batched command-line caller: the reference CLI's build and
query subcommands (tools/rbe_main.cpp:103-211) over the HBM-resident index -- same output line
format, same exit codes, per-batch latency report."""
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle import gen_queries
from tests.test_rbee_build import corpus, write_rbee

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1802_06466_b200", "_lib", "rbe-cuda")


def run(*args):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True)


def test_cli_usage_and_errors(tmp_path):
    assert run("--help").returncode == 0
    r = run()
    assert r.returncode == 2
    r = run("query", "--bogus", "1")
    assert r.returncode == 2 and "unknown option: --bogus" in r.stderr
    r = run("query", "--index", tmp_path / "missing.rbei", "--queries", tmp_path / "q.rbee")
    assert r.returncode == 1 and "error: cannot open index:" in r.stderr
    r = run("query", "--index", "x", "--queries", "y", "--n", "0")
    assert r.returncode == 2 and "--n: expected a positive integer" in r.stderr
    r = run("build", "--embeddings", tmp_path / "missing.rbee", "--output", tmp_path / "o.rbei")
    assert r.returncode == 1 and "error: cannot open embeddings file:" in r.stderr
    r = run("frobnicate")
    assert r.returncode == 2


@pytest.mark.gpu
def test_cli_build_and_query_match_reference(ref, tmp_path):
    dim, kp, rw, P, n_docs, n = 128, 3, True, 4, 30_000, 25
    ids, words, _ = corpus(dim, kp, n_docs, 11)
    write_rbee(tmp_path / "docs.rbee", dim, kp, rw, ids, words, np.zeros(n_docs, np.float32))
    r = run("build", "--embeddings", tmp_path / "docs.rbee", "--output", tmp_path / "ix.rbei", "--partitions", P)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith(f"keywords={n_docs} partitions={P} plane_bytes_per_keyword=48 ")
    theirs = ref.build_index(dim, kp, rw, P, words, ids)
    theirs.save(tmp_path / "ref.rbei")
    assert (tmp_path / "ix.rbei").read_bytes() == (tmp_path / "ref.rbei").read_bytes()

    Q = 7
    qw = gen_queries(0x0E1, Q, dim, kp)  # [Q][qp][wpp]
    write_rbee(tmp_path / "q.rbee", dim, kp, rw, np.arange(Q, dtype=np.uint64), qw, np.zeros(Q, np.float32))
    r = run("query", "--index", tmp_path / "ix.rbei", "--queries", tmp_path / "q.rbee", "--n", n, "--batch-size", 3,
            "--devices", "0,0")
    assert r.returncode == 0, r.stderr
    geo = (1, 256, 256, 1)  # auto blocks: ceil(7500 / 65536) = 1
    want, _ = ref.load_index(tmp_path / "ref.rbei").search(qw, geo, n)
    lines = [f"{q}\t{i}\t{float(s):.9g}" for q in range(Q) for s, i, _ in want[q]]
    assert r.stdout.splitlines() == lines
    assert f"queries={Q} latency_mean_ms=" in r.stderr
    assert "batches=3 batch_size=3 batch_latency_mean_ms=" in r.stderr and "batch_latency_p99_ms=" in r.stderr
