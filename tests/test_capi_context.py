"""cft_init / cft_destroy (SURVEY §8(b) context entry points): on a B200 cft_init binds the
device; a device that does not exist (or no GPU at all, as in this container) is an error
status with a message, never a crash; cft_destroy clears the thread's error state."""
import pytest

torch = pytest.importorskip("torch")


def test_init_refuses_a_missing_device():
    from paper_2605_21177_b200 import _native as N
    assert N.lib.cft_init(1 << 20) != N.CFT_OK
    msg = N.lib.cft_last_error().decode()
    assert "no such CUDA device" in msg or "cudaGetDeviceCount" in msg
    assert N.lib.cft_destroy() == N.CFT_OK
    assert N.lib.cft_last_error() == b""


@pytest.mark.gpu
def test_init_binds_the_b200(cuda):
    from paper_2605_21177_b200 import _native as N
    assert N.lib.cft_init(0) == N.CFT_OK, N.lib.cft_last_error()
    assert N.lib.cft_destroy() == N.CFT_OK


def test_nccl_and_state_entries_refuse_bad_arguments_without_crashing():
    """Argument checks of the communicator / state-move entries run before any CUDA or NCCL call
    (CPU: no device needed)."""
    import ctypes as C
    from paper_2605_21177_b200 import _native as N
    assert N.lib.cft_allreduce_f32(None, 4, None, None) != N.CFT_OK
    assert b"null communicator" in N.lib.cft_last_error()
    N.lib.cft_comm_nccl_create.argtypes = [C.c_void_p, C.c_void_p]
    assert N.lib.cft_comm_nccl_create(None, None) != N.CFT_OK
    assert b"null communicator" in N.lib.cft_last_error()
    assert N.lib.cft_states_prefetch(None, 4, N.CFT_F32, None, None, None, None, None, None) != N.CFT_OK
    assert b"null buffer" in N.lib.cft_last_error()
    assert N.lib.cft_states_offload(None, None, None, -1, N.CFT_F32, None, None, None, None) != N.CFT_OK
    assert b"negative element count" in N.lib.cft_last_error()
    assert N.lib.cft_norm_dgamma_slice(N.CFT_F32, None, None, None, None, 4, 8, 5, 9, None, 0,
                                       None) != N.CFT_OK
    assert b"out of bounds" in N.lib.cft_last_error()
