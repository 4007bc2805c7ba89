"""The reference's acceptance criterion 3 (tests/acceptance.cpp:254-296) on the native host
planner: a schedule dry run's peak memory equals the 2M + 16M/K closed form exactly, for a
7e9-element virtual tensor at K in {1, 4, 8, 64}, with the K=1 byte decomposition and the K=8
figure pinned as the reference pins them.  CPU only (no device): the accounting is host C++
(csrc/host/plan_capi.cpp cft_simulate_memory_trace / cft_model_peak_bytes)."""
import pytest

from paper_2605_21177_b200.plan import (ScheduleConfig, TensorInfo, model_peak_bytes, partition,
                                        simulate_memory_trace)


def test_simulated_peak_matches_closed_form():
    big = TensorInfo(0, "virtual", 7_000_000, 1000, storage_precision=2)
    m = big.rows * big.cols
    for K in (1, 4, 8, 64):
        plan = partition([big], K)
        trace = simulate_memory_trace([big], plan, ScheduleConfig(K=K, T=1, total_steps=2 * K))
        predicted = 2.0 * m + 16.0 * m / K
        assert max(trace) == predicted, (K, max(trace), predicted)
        assert model_peak_bytes(m, K) == predicted
        if K == 1:  # 18 B/elem: 2 resident + 4 grad + 12 master / m / v
            assert max(trace) == 18.0 * m == 126e9
        if K == 8:
            assert max(trace) == 28e9


@pytest.mark.parametrize("K,T,prefetch,bw,act", [(3, 2, True, 100, 0), (3, 2, False, 100, 0),
                                                  (5, 1, True, 0, 4096), (2, 3, True, 7, 64)])
def test_memory_trace_matches_reference_dry_run(K, T, prefetch, bw, act):
    """Against the reference's own simulate_memory_trace (oracle/_ref) for prefetching and
    bandwidth-limited schedules (the in-flight windows of schedule.cpp:129-135) and mixed
    storage precisions: every step's total, byte for byte."""
    from oracle import ref
    if not ref.available:
        pytest.skip("oracle/_ref not built")
    tensors = [(0, 8, 4, 2), (1, 4, 4, 4), (2, 6, 3, 1), (3, 5, 1, 8)]
    infos = [TensorInfo(i, f"t{i}", r, c, storage_precision=sp) for i, r, c, sp in tensors]
    plan = partition(infos, K)
    steps = 4 * K * T
    cfg = ScheduleConfig(K=plan.K, T=T, total_steps=steps, prefetch=prefetch,
                         bandwidth_bytes_per_step=bw)
    ours = simulate_memory_trace(infos, plan, cfg, act)
    want = ref.simulate_memory_trace(tensors, K, T, steps, prefetch, bw, act)
    assert ours == want


def test_model_peak_bytes_rejects_bad_arguments():
    from paper_2605_21177_b200._native import CftError
    with pytest.raises(CftError):
        model_peak_bytes(0, 4)
    with pytest.raises(CftError):
        model_peak_bytes(10, 0)
