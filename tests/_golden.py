"""Replays tests/golden/*.npz (outputs of the reference itself) through any
implementation of ok_sparse_allreduce."""
import glob
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def cases():
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(HERE, "*.npz")))


def load(name):
    return dict(np.load(os.path.join(HERE, name)))


def check_step(fx, t, P, got_u_idx, got_u_val, got_indexes, got_sel, got_ledger=None, got_states=None):
    """Assert one iteration equals the reference's recorded result."""
    assert np.array_equal(got_u_idx, fx[f"u_idx_t{t}"]), f"t={t}: u indices differ"
    assert np.array_equal(got_u_val, fx[f"u_val_t{t}"]), f"t={t}: u values differ"
    for r in range(P):
        assert np.array_equal(got_indexes[r], fx[f"ix_t{t}_r{r}"]), f"t={t} rank {r}: indexes differ"
    assert list(got_sel) == list(fx[f"sel_t{t}"]), f"t={t}: local_selected differ"
    if got_ledger is not None:
        assert np.array_equal(got_ledger, fx[f"ledger_t{t}"]), f"t={t}: ledger differs"
    if got_states is not None:
        assert np.array_equal(got_states, fx[f"state_t{t}"]), f"t={t}: OkState differs"
