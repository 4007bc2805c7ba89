"""NCCL behind the C ABI's communicator (cft_allreduce_f32, cft_comm_nccl_create),
on the one GPU a box has: a one-rank communicator made by the host (ncclGetUniqueId +
ncclCommInitRank through ctypes, as a C++ host would), every collective the data-parallel step
issues queued on a stream and checked, and cft_engine_step_dp with the NCCL communicator equal
bit for bit to the plain step (world 1: grad_scale 1).  Multi-rank NCCL needs one GPU per rank
(NCCL rejects two ranks on one device); the exchange protocols themselves are covered with
host callbacks across two processes (test_gpu_capi_dp.py) and with gloo (test_dp.py)."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


class NcclUniqueId(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]


STREAM = C.c_void_p
AR = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, STREAM)
RS = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, STREAM)
AG = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, STREAM)
BAR = C.CFUNCTYPE(C.c_int, C.c_void_p, STREAM)


class CftComm(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("world", C.c_int32), ("rank", C.c_int32),
                ("all_reduce", AR), ("reduce_scatter", RS), ("all_gather", AG), ("barrier", BAR)]


@pytest.fixture(scope="module")
def nccl_comm(cuda):
    torch.zeros(1, device="cuda")  # context up before NCCL
    nccl = C.CDLL("libnccl.so.2", mode=C.RTLD_GLOBAL)
    uid = NcclUniqueId()
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
    comm = C.c_void_p()
    assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
    yield comm
    nccl.ncclCommDestroy(comm)


def _lib():
    from paper_2605_21177_b200._native import lib
    lib.cft_allreduce_f32.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
    lib.cft_comm_nccl_create.argtypes = [C.c_void_p, C.POINTER(CftComm)]
    lib.cft_comm_nccl_destroy.argtypes = [C.POINTER(CftComm)]
    lib.cft_engine_step_dp.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(CftComm)]
    return lib


def test_allreduce_and_every_collective_of_the_step(nccl_comm):
    lib = _lib()
    s = torch.cuda.Stream()
    x = torch.randn(4097, device="cuda")
    ref = x.clone()
    assert lib.cft_allreduce_f32(x.data_ptr(), x.numel(), nccl_comm, s.cuda_stream) == 0
    s.synchronize()
    assert torch.equal(x, ref)  # one rank: the sum is the buffer
    assert lib.cft_allreduce_f32(x.data_ptr(), 4, None, s.cuda_stream) != 0  # null comm: error
    assert b"null communicator" in lib.cft_last_error()

    comm = CftComm()
    assert lib.cft_comm_nccl_create(nccl_comm, C.byref(comm)) == 0
    try:
        assert (comm.world, comm.rank) == (1, 0)
        for dt, tdt in ((0, torch.float32), (2, torch.float64), (1, torch.bfloat16)):
            a = torch.randn(1000, device="cuda").to(tdt)
            a0 = a.clone()
            assert comm.all_reduce(comm.ctx, a.data_ptr(), a.numel(), dt, s.cuda_stream) == 0
            out = torch.empty_like(a)
            assert comm.reduce_scatter(comm.ctx, a.data_ptr(), out.data_ptr(), a.numel(), dt,
                                       s.cuda_stream) == 0
            assert comm.all_gather(comm.ctx, out.data_ptr(), out.numel(), dt, s.cuda_stream) == 0
            assert comm.barrier(comm.ctx, s.cuda_stream) == 0
            s.synchronize()
            assert torch.equal(a, a0) and torch.equal(out, a0)
    finally:
        lib.cft_comm_nccl_destroy(C.byref(comm))
    assert comm.ctx is None


def test_step_dp_over_nccl_equals_the_plain_step(nccl_comm):
    from paper_2605_21177_b200.engine import ChunkEngine, Model, TrainOptions
    from paper_2605_21177_b200.plan import ScheduleConfig
    lib = _lib()
    rng = np.random.default_rng(5)
    m = Model(loss="half_sq").add_linear(12, 16).add_tanh().add_linear(16, 3)
    init = rng.uniform(-0.4, 0.4, m.num_params())
    batches = [{"x": rng.uniform(-1, 1, (6, 12)), "target": rng.uniform(-1, 1, (6, 3))}
               for _ in range(3)]
    steps = 9
    opts = TrainOptions(schedule=ScheduleConfig(K=3, T=2, total_steps=steps), dtype="fp64")
    plain = ChunkEngine(m, init, 6, opts)
    dp = ChunkEngine(m, init, 6, opts)
    comm = CftComm()
    assert lib.cft_comm_nccl_create(nccl_comm, C.byref(comm)) == 0
    try:
        sp = [plain.stage(b, device=True) for b in batches]
        sd = [dp.stage(b, device=True) for b in batches]
        for t in range(steps):
            plain.step([sp[t % 3]])
            assert lib.cft_engine_step_dp(dp._h, C.byref(sd[t % 3]), C.byref(comm)) == 0, \
                lib.cft_last_error()
        plain.finish()
        dp.finish()
    finally:
        lib.cft_comm_nccl_destroy(C.byref(comm))
    assert np.array_equal(plain.params(), dp.params())
    assert np.array_equal(plain.trajectory()["loss"], dp.trajectory()["loss"])
