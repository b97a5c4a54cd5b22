"""CPU checks of the multi-GPU iteration pipeline's host logic
(paper_2310_11365_b200/sharded_pipeline.py): slice ownership, the exchange
block layout, and that the end-of-run merge takes every trace entry from the
rank whose units wrote it.  The unit write pattern restated here follows
csrc/pipeline.cu (match part of unit (k, n): macro/micro[k][n],
cache/coarse_status/match_status[k][n-1], raw[k-1][n-1]; fine part:
fine_stats/fine_counts/bad[k][n]; unit (k, 0): macro/micro[k][0]; the
prologue: row 0)."""

import numpy as np
import pytest

from paper_2310_11365_b200 import sharded_pipeline as SP


def _writes(r, G, N, K):
    """(array, row, index) entries rank r's units and prologue write."""
    Ng = N // G
    out = set()
    for n in SP.owned_boundaries(r, Ng, G, N):
        # prologue: coarse row 0 everywhere (redundant), lift of owned boundaries
        out.add(("macro", 0, n))
        out.add(("micro", 0, n))
        if n >= 1:
            out.add(("match_status", 0, n - 1))
        for k in range(K + 1):
            if k >= 1 and n >= 1:
                out |= {("macro", k, n), ("micro", k, n), ("cache", k, n - 1), ("coarse_status", k, n - 1),
                        ("match_status", k, n - 1), ("raw", k - 1, n - 1)}
            elif k >= 1:
                out |= {("macro", k, 0), ("micro", k, 0)}
            if k < K and n < N:
                out |= {("fine_stats", k, n), ("bad", k, n)}
    return out


@pytest.mark.parametrize("G,N,K", [(2, 8, 3), (4, 16, 5), (8, 64, 5), (3, 9, 9), (1, 5, 2)])
def test_merge_takes_each_entry_from_its_writer(G, N, K):
    Ng = N // G
    shapes = {"macro": (K + 1, N + 1), "micro": (K + 1, N + 1), "fine_stats": (K, N), "bad": (K, N),
              "raw": (K, N), "cache": (K + 1, N), "coarse_status": (K + 1, N), "match_status": (K + 1, N)}
    kinds = {"macro": "boundary", "micro": "boundary", "fine_stats": "slice", "bad": "slice", "raw": "shifted",
             "cache": "shifted", "coarse_status": "shifted", "match_status": "shifted"}
    writes = [_writes(r, G, N, K) for r in range(G)]
    for name, shape in shapes.items():
        parts = []
        for r in range(G):
            a = np.full(shape, -1.0)  # never written by rank r
            for (arr, k, i) in writes[r]:
                if arr == name:
                    a[k, i] = r
            parts.append(a)
        merged = SP.merge_rows(parts, Ng, G, N, kinds[name])
        for k in range(shape[0]):
            for i in range(shape[1]):
                writers = {r for r in range(G) if (name, k, i) in writes[r]}
                if name == "cache" and k == 0:
                    continue  # the prologue's coarse row: every rank (redundant), not in _writes
                if name == "coarse_status" and k == 0:
                    continue
                if not writers:
                    continue  # never written (e.g. raw has no row for k = K)
                assert merged[k, i] in writers, (name, k, i, merged[k, i], writers)


def test_every_unit_is_owned_once():
    for G, N in ((2, 8), (4, 16), (8, 512), (3, 9)):
        Ng = N // G
        seen = [n for r in range(G) for n in SP.owned_boundaries(r, Ng, G, N)]
        assert seen == list(range(N + 1))
        assert all(SP.owner(n, Ng, G) == r for r in range(G) for n in SP.owned_boundaries(r, Ng, G, N))


def test_exchange_layout_is_aligned_and_disjoint():
    L = SP.exchange_layout(512, 5, 100_000)
    spans = []
    for name in ("flags", "macro", "fine_stats", "fine_counts", "fine"):
        off, count, dtype = L[name]
        assert off % 256 == 0
        size = count * (4 if "int32" in str(dtype) else 8)
        spans.append((off, off + size))
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 <= b0
    assert spans[-1][1] <= L["_bytes"]
    assert L["fine"][1] == 2 * 512 * 100_000
