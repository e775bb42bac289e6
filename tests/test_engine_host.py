"""Host-side control of the device engine that needs no GPU: the run-ahead batch sizing."""

from paper_2305_19013_b200.engine import DeviceEngine


def snap(k, rho, tol_abs=1e-8):
    return {"live": 1, "status": 0, "k_done": k, "last_rho": rho, "tol_abs": tol_abs}


def test_batch_size_falls_back_to_lookahead():
    assert DeviceEngine._batch_size(8, [], 5) == 8
    assert DeviceEngine._batch_size(8, [snap(3, 1.0)], 5) == 8
    # no decay (stagnation or growth): keep doubling
    assert DeviceEngine._batch_size(16, [snap(3, 1.0), snap(5, 1.0)], 9) == 16
    assert DeviceEngine._batch_size(16, [snap(3, 1.0), snap(5, 2.0)], 9) == 16


def test_batch_size_follows_predicted_remaining_iterations():
    # residual falls by 5x per iteration: from 2e-4 to 1e-8 takes log(5e-5) / log(0.2) = 6.15 more
    # iterations after k = 10; with 11..12 already queued (k_next = 13) -> ceil(1.25 * 6.15) + 2 - 2 = 8
    seen = [snap(9, 1e-3), snap(10, 2e-4)]
    assert DeviceEngine._batch_size(16, seen, 13) == 8
    # capped by the look-ahead, never below 1
    assert DeviceEngine._batch_size(2, seen, 13) == 2
    assert DeviceEngine._batch_size(16, seen, 40) == 1
    # below tolerance at the snapshot (the stop test then has already cleared the live flag): the margin only
    assert DeviceEngine._batch_size(16, [snap(9, 1e-7), snap(10, 1e-9)], 11) == 2
