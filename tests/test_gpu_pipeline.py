"""The pipelined Alg. 5 loop (cf.auto_latent_factors): block l+1 is queued
ahead of block l's stop decision only when that decision cannot end the
scan (fewer than patience - 1 stale blocks), so no QB block is computed
past the stop, and the trace equals the sequential loop's."""
from __future__ import annotations

import pytest

import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(gpu):
    import paper_2009_02251_b200 as P
    return P


@pytest.mark.parametrize("patience", [1, 2, 3])
def test_no_block_past_the_stop(P, monkeypatch, patience):
    from paper_2009_02251_b200 import cf
    train, val, _ = inputs.group_model(300, 240, 6, 0.6, seed=9)
    A = P.SparseRatings(train, 1.0, 5.0)
    real = cf.qb_pass_blocks
    made = []

    def counting(*a, **kw):
        for s in real(*a, **kw):
            made.append(s.rank)
            yield s

    monkeypatch.setattr(cf, "qb_pass_blocks", counting)
    runs = {}
    for pipe in (True, False):
        monkeypatch.setattr(cf, "PIPELINE", pipe)
        made.clear()
        f, trace = P.auto_latent_factors(A, val, block_size=3, passes=6, patience=patience, seed=1)
        runs[pipe] = (f.k, [(e.k, e.mae) for e in trace], list(made))
    for pipe, (k, trace, blocks) in runs.items():
        assert blocks == [kk for kk, _ in trace], f"pipeline={pipe}: computed {blocks}, scored {trace}"
    assert runs[True][:2] == runs[False][:2]
