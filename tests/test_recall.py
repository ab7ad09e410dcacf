"""Recall of the lossy scan against the Appendix A model (PAPER.md:327-329,
src/analysis.cpp:143-184): with queue length 1 each logical thread keeps only its best item,
so recall@N of a search with I items per thread is the expected fraction of the N relevant
(truly top-N) keywords that sit alone at the top of their thread.  The device's lossless
result (one item per logical thread) is the ground truth; the reference's own
expected_recall (compiled from its sources) is the prediction."""
import math

import numpy as np
import pytest

from oracle.oracle import gen_queries

pytestmark = pytest.mark.gpu


def geometry(rbe, tpb, ipt, count):
    g = rbe.ScanGeometry()
    g.threads_per_block, g.items_per_thread, g.queue_length = tpb, ipt, 1
    g.blocks = -(-count // (tpb * ipt))
    return g


def measured_recall(rbe, dix, qs, count, n, ipt):
    exact = dix.search_words(qs, geometry(rbe, 256, 1, count), n)[1]  # ids: one item per thread, no loss
    lossy = dix.search_words(qs, geometry(rbe, 256, ipt, count), n)[1]
    return [len(set(exact[q].tolist()) & set(lossy[q].tolist())) / n for q in range(qs.shape[0])]


@pytest.mark.parametrize("ipt", [256, 64])
def test_recall_matches_appendix_a(rbe, ref, ipt):
    C, n, Q = 4_000_000, 1000, 64
    dix = rbe.DeviceIndex.synthetic(128, 3, True, C, 1, 0xD0C5)
    qs = gen_queries(0x5EC, Q, 128, 3)
    r = measured_recall(rbe, dix, qs, C, n, ipt)
    want, _ = ref.expected_recall(C, n, ipt)
    got = float(np.mean(r))
    se = math.sqrt(want * (1 - want) / (Q * n))
    assert abs(got - want) <= 4 * se + 2e-3, (got, want, se)
