"""C5 sweep (BASELINE configs[4]): micro-batches 1..16 x workers {2,4,8} on
the product plan layer — closed-form and measured version difference, the
N = 1 domain error and the slot-model idle fraction — against the oracle
restatement (ledger.cpp:121-147, metrics.cpp:71-72)."""
import numpy as np
import pytest

from oracle import pipesim_np as O
from tools import sweep


@pytest.mark.parametrize("W", [2, 4, 8])
def test_sweep_plan_cells_match_oracle(W):
    for N in range(1, 17):
        rec = sweep.plan_cell(W, N)
        if N == 1:
            assert "domain_error" in rec and "micro_batches" in rec["domain_error"]
            with pytest.raises(ValueError):
                O.closed_form_v(W, N)
            continue
        M = 2 * (W + N)
        grid = O.build_schedule(W, N, M)
        led = O.assign_versions(grid, W, N, M)
        assert rec["closed_form_v"] == O.closed_form_v(W, N)
        assert rec["measured_v"] == O.measure_version_difference(led["update_source"], W, N, M)
        assert rec["measured_v"] == (W - 1) // (N + 1) + 1
        assert rec["horizon"] == grid.shape[1]
        idle = np.sum(grid[:, :, 0] == 0) / (W * grid.shape[1])
        assert rec["slot_idle_fraction"] == pytest.approx(idle, abs=0)


def test_known_divergent_cells():
    # closed form != measured at (8,2) and (8,3)
    assert (sweep.plan_cell(8, 2)["closed_form_v"], sweep.plan_cell(8, 2)["measured_v"]) == (4, 3)
    assert (sweep.plan_cell(8, 3)["closed_form_v"], sweep.plan_cell(8, 3)["measured_v"]) == (3, 2)
