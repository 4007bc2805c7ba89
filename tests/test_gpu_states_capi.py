"""cft_states_prefetch / cft_states_offload (the reference's load_to_device /
offload_to_host, src/optimizer.cpp:101-122, whose round trip is bit-identical,
tests/acceptance.cpp:435-493): a chunk's [master | m | v] block moves between pinned host memory
and a device slot on a stream, ordered by events; a rotation driven by the C-ABI scheduler
(cft_scheduler_*) with these moves leaves every chunk's host block holding exactly the updates
made while it was resident; an unpinned host block is refused."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _moves():
    from paper_2605_21177_b200 import _native as N

    def prefetch(block, n, dt, dev, stream, wait=None, done=None):
        N.check(N.lib.cft_states_prefetch(block.data_ptr(), n, dt, dev[0].data_ptr(),
                                          dev[1].data_ptr(), dev[2].data_ptr(), stream.cuda_stream,
                                          wait.cuda_event if wait else None,
                                          done.cuda_event if done else None), "prefetch")

    def offload(dev, n, dt, block, stream, wait=None, done=None):
        N.check(N.lib.cft_states_offload(dev[0].data_ptr(), dev[1].data_ptr(), dev[2].data_ptr(), n,
                                         dt, block.data_ptr(), stream.cuda_stream,
                                         wait.cuda_event if wait else None,
                                         done.cuda_event if done else None), "offload")
    return N, prefetch, offload


def _event(stream):
    """A torch event whose CUDA handle exists (torch creates it at the first record), so the
    library can record it as done_event."""
    e = torch.cuda.Event()
    e.record(stream)
    return e


@pytest.mark.parametrize("tdt,dt", [(torch.float32, 0), (torch.float64, 2)])
def test_round_trip_is_bit_identical(cuda, tdt, dt):
    N, prefetch, offload = _moves()
    n = 100_003
    block = torch.randn(3 * n, dtype=tdt).pin_memory()
    back = torch.zeros(3 * n, dtype=tdt).pin_memory()
    dev = [torch.empty(n, dtype=tdt, device="cuda") for _ in range(3)]
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    loaded = _event(h2d)
    prefetch(block, n, dt, dev, h2d, done=loaded)
    offload(dev, n, dt, back, d2h, wait=loaded)  # the D2H stream waits for the H2D event only
    d2h.synchronize()
    assert torch.equal(back, block)
    for k in range(3):
        assert torch.equal(dev[k].cpu(), block[k * n:(k + 1) * n])


def test_unpinned_and_bad_arguments_are_refused(cuda):
    N, prefetch, offload = _moves()
    n = 16
    dev = [torch.empty(n, device="cuda") for _ in range(3)]
    s = torch.cuda.Stream()
    with pytest.raises(N.CftError, match="not pinned"):
        prefetch(torch.zeros(3 * n), n, 0, dev, s)
    with pytest.raises(N.CftError, match="fp32 or fp64"):
        prefetch(torch.zeros(3 * n).pin_memory(), n, 1, dev, s)


def test_rotation_driven_by_the_c_abi_scheduler(cuda):
    """Three chunks of different sizes, K = 3, T = 2, prefetch on: the scheduler's physical
    moves (schedule.cpp:17-135) are carried out with cft_states_*; while a chunk is resident its
    device master gets +1 per step.  Each host block must end with master = initial + (number of
    steps the chunk was active), m and v untouched."""
    N, prefetch, offload = _moves()
    from paper_2605_21177_b200 import plan as P
    infos = [P.TensorInfo(0, "a", 8, 4), P.TensorInfo(1, "b", 6, 5)]
    plan = P.partition(infos, 3)
    sizes = [plan.chunks[c].elements for c in range(3)]
    steps, T = 12, 2
    blocks = [torch.arange(3 * n, dtype=torch.float32).pin_memory() for n in sizes]
    initial = [b.clone() for b in blocks]
    slots = [[torch.empty(max(sizes), device="cuda") for _ in range(3)] for _ in range(3)]
    owner = [-1, -1, -1]  # chunk held by each device slot
    compute, h2d, d2h = torch.cuda.current_stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ready = [_event(h2d) for _ in range(3)]
    freed = [_event(d2h) for _ in range(3)]
    active_steps = [0, 0, 0]
    sched = P.RotationScheduler(P.ScheduleConfig(K=3, T=T, total_steps=steps, prefetch=True), plan)

    def load(c):
        if c in owner:
            return owner.index(c)
        s = owner.index(-1)
        dev = [t[:sizes[c]] for t in slots[s]]
        prefetch(blocks[c], sizes[c], 0, dev, h2d, wait=freed[s], done=ready[s])
        owner[s] = c
        return s

    for t in range(steps):
        active = sched.step_begin()
        for c in (sched.last_load, sched.last_prefetch):
            if c >= 0:
                load(c)
        s = load(active)
        compute.wait_event(ready[s])
        slots[s][0][:sizes[active]].add_(1.0)  # the "update" of the resident master
        active_steps[active] += 1
        done = torch.cuda.Event()
        done.record(compute)
        sched.step_end()
        off = sched.last_offload
        if off >= 0:
            so = owner.index(off)
            offload([x[:sizes[off]] for x in slots[so]], sizes[off], 0, blocks[off], d2h, wait=done,
                    done=freed[so])
            owner[so] = -1
    for c in sched.finish():
        if c in owner:
            so = owner.index(c)
            offload([x[:sizes[c]] for x in slots[so]], sizes[c], 0, blocks[c], d2h,
                    wait=torch.cuda.current_stream().record_event(), done=freed[so])
            owner[so] = -1
    torch.cuda.synchronize()
    for c in range(3):
        n = sizes[c]
        want = initial[c].clone()
        want[:n] += active_steps[c]
        assert torch.equal(blocks[c], want), c
    assert sum(active_steps) == steps and all(a > 0 for a in active_steps)
