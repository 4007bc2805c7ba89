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
