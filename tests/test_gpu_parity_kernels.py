"""The parity-level boundary: the twelve `cft_kernels_*` entry points (the `Backend::cuda` a
maintainer adds to the reference's dispatch, src/kernels.cpp:37-68)
called through the C ABI with host double* buffers, against the UNMODIFIED reference kernels
(oracle/_ref, Backend::serial) on identical inputs.  Bit-identical for every kernel, tanh
included (the CUDA kernel restates glibc's tanh / expm1 operation by operation).  Includes the reference's own edge cases:
empty ranges leave buffers untouched (tests/test_kernels.cpp:205-219), out-of-range and
duplicate tokens in the embedding scatter (tests/test_ops.cpp:134-178), accumulate semantics.

Also runs the reference's unit-test suites and acceptance run against this backend, when
oracle/ref_cuda/Makefile built them here (they travel to the GPU box in oracle/_ref/cuda)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D = C.POINTER(C.c_double)


@pytest.fixture(scope="module")
def libs(cuda):
    from oracle import ref as R
    if not R.available:
        pytest.skip("oracle/_ref (the reference library) not built")
    from paper_2605_21177_b200 import _native as N
    R.set_backend(False)  # Backend::serial: the reference's per-element order
    yield N.lib, R.REF
    R.set_backend(True)


@pytest.fixture(autouse=True)
def _clear_status(libs):
    libs[0].cft_last_status()  # reading resets the thread's sticky status


def d(a):
    return a.ctypes.data_as(D)


def i(a):
    return a.ctypes.data_as(C.c_void_p)


def status(lib):
    st = lib.cft_last_status()
    assert st == 0, lib.cft_last_error()


def rnd(rng, *shape):
    return rng.uniform(-2.0, 2.0, shape)


def same(a, b):
    assert a.shape == b.shape and a.tobytes() == b.tobytes(), np.max(np.abs(a - b))


@pytest.mark.parametrize("batch,in_dim,out_dim,bias", [(1, 2, 2, True), (7, 33, 19, False),
                                                       (64, 128, 96, True)])
def test_linear_forward_dinput_bitwise(libs, batch, in_dim, out_dim, bias):
    lib, ref = libs
    rng = np.random.default_rng(batch * 1000 + in_dim)
    x, w, b = rnd(rng, batch, in_dim), rnd(rng, out_dim, in_dim), rnd(rng, out_dim)
    y_ref, y = np.full((batch, out_dim), 7.0), np.full((batch, out_dim), 7.0)
    ref.ref_linear_forward(i(x), batch, in_dim, i(w), out_dim, i(b) if bias else None, i(y_ref))
    lib.cft_kernels_linear_forward(d(x), batch, in_dim, d(w), out_dim, d(b) if bias else None, d(y))
    status(lib)
    same(y, y_ref)
    dy = rnd(rng, batch, out_dim)
    dx0 = rnd(rng, batch, in_dim)  # += semantics: accumulate onto a non-zero buffer
    dx_ref, dx = dx0.copy(), dx0.copy()
    ref.ref_linear_dinput(i(dy), batch, out_dim, i(w), in_dim, i(dx_ref))
    lib.cft_kernels_linear_dinput(d(dy), batch, out_dim, d(w), in_dim, d(dx))
    status(lib)
    same(dx, dx_ref)


def test_linear_forward_hand_case(libs):
    """tests/test_kernels.cpp:44-57: W=[[1,2],[3,4]], x=[1,1], b=[10,20] -> y=[13,27]."""
    lib, _ = libs
    x, w, b = np.ones(2), np.array([1.0, 2.0, 3.0, 4.0]), np.array([10.0, 20.0])
    y = np.zeros(2)
    lib.cft_kernels_linear_forward(d(x), 1, 2, d(w), 2, d(b), d(y))
    status(lib)
    assert y.tolist() == [13.0, 27.0]


@pytest.mark.parametrize("rb,re", [(0, 19), (3, 11), (18, 19), (5, 5)])
def test_linear_dweight_dbias_slices_bitwise(libs, rb, re):
    lib, ref = libs
    rng = np.random.default_rng(rb * 31 + re)
    batch, out_dim, in_dim = 13, 19, 41
    dy, x = rnd(rng, batch, out_dim), rnd(rng, batch, in_dim)
    dw0 = rnd(rng, max(re - rb, 1), in_dim)
    dw_ref, dw = dw0.copy(), dw0.copy()
    ref.ref_linear_dweight(i(dy), batch, out_dim, i(x), in_dim, rb, re, i(dw_ref))
    lib.cft_kernels_linear_dweight(d(dy), batch, out_dim, d(x), in_dim, rb, re, d(dw))
    status(lib)
    same(dw, dw_ref)
    if re == rb:  # empty range: the buffer is untouched (tests/test_kernels.cpp:205-219)
        same(dw, dw0)
    db0 = rnd(rng, max(re - rb, 1))
    db_ref, db = db0.copy(), db0.copy()
    ref.ref_linear_dbias(i(dy), batch, out_dim, rb, re, i(db_ref))
    lib.cft_kernels_linear_dbias(d(dy), batch, out_dim, rb, re, d(db))
    status(lib)
    same(db, db_ref)


def test_embedding_gather_scatter_bitwise(libs):
    lib, ref = libs
    rng = np.random.default_rng(5)
    vocab, dim, positions = 37, 24, 60
    table = rnd(rng, vocab, dim)
    tok = rng.integers(0, vocab, positions).astype(np.int32)
    tok[:6] = [3, 3, 3, 36, 0, 36]  # duplicates accumulate
    y_ref, y = np.zeros((positions, dim)), np.zeros((positions, dim))
    ref.ref_embedding_gather(i(table), dim, i(tok), positions, i(y_ref))
    lib.cft_kernels_embedding_gather(d(table), dim, i(tok), positions, d(y))
    status(lib)
    same(y, y_ref)
    dy = rnd(rng, positions, dim)
    for rb, re in [(0, vocab), (3, 4), (10, 30), (36, 37), (20, 20)]:
        dt0 = rnd(rng, max(re - rb, 1), dim)
        dt_ref, dt = dt0.copy(), dt0.copy()
        m_ref = ref.ref_embedding_scatter(i(dy), dim, i(tok), positions, rb, re, i(dt_ref))
        m = lib.cft_kernels_embedding_scatter(d(dy), dim, i(tok), positions, rb, re, d(dt))
        status(lib)
        assert m == m_ref
        same(dt, dt_ref)


def test_embedding_scatter_out_of_range_and_duplicates(libs):
    """tests/test_ops.cpp:134-178 at the kernel level: tokens outside [rb, re) contribute
    nothing, duplicates of an in-range row add ([2, 2] for two unit rows)."""
    lib, _ = libs
    dim = 2
    tok = np.array([1, 1, 5, -3, 9], np.int32)
    dy = np.ones((5, dim))
    dt = np.zeros((3, dim))  # rows [0, 3)
    m = lib.cft_kernels_embedding_scatter(d(dy), dim, i(tok), 5, 0, 3, d(dt))
    status(lib)
    assert m == 2
    assert dt.tolist() == [[0.0, 0.0], [2.0, 2.0], [0.0, 0.0]]


def test_embedding_gather_negative_id_reads_nothing(libs):
    """A negative id (the reference's ops layer throws before its kernel sees one,
    ops.cpp:53-54) produces a zero row instead of a read before the table."""
    lib, _ = libs
    table = np.arange(8.0).reshape(4, 2)
    tok = np.array([2, -1, 0], np.int32)
    y = np.full((3, 2), 9.0)
    lib.cft_kernels_embedding_gather(d(table), 2, i(tok), 3, d(y))
    status(lib)
    assert y.tolist() == [[4.0, 5.0], [0.0, 0.0], [0.0, 1.0]]


@pytest.mark.parametrize("batch,dim", [(1, 3), (9, 64), (33, 257)])
def test_layernorm_kernels_bitwise(libs, batch, dim):
    lib, ref = libs
    rng = np.random.default_rng(batch + dim)
    x, g, b = rnd(rng, batch, dim), rnd(rng, dim), rnd(rng, dim)
    outs_ref = [np.zeros((batch, dim)), np.zeros(batch), np.zeros(batch)]
    outs = [np.zeros((batch, dim)), np.zeros(batch), np.zeros(batch)]
    ref.ref_layernorm_forward(i(x), batch, dim, i(g), i(b), C.c_double(1e-5), *[i(o) for o in outs_ref])
    lib.cft_kernels_layernorm_forward(d(x), batch, dim, d(g), d(b), 1e-5, *[d(o) for o in outs])
    status(lib)
    for a, r in zip(outs, outs_ref):
        same(a, r)
    y, mean, istd = outs_ref
    dy = rnd(rng, batch, dim)
    dx0 = rnd(rng, batch, dim)
    dx_ref, dx = dx0.copy(), dx0.copy()
    ref.ref_layernorm_dinput(i(dy), i(x), i(mean), i(istd), i(g), batch, dim, i(dx_ref))
    lib.cft_kernels_layernorm_dinput(d(dy), d(x), d(mean), d(istd), d(g), batch, dim, d(dx))
    status(lib)
    same(dx, dx_ref)
    for rb, re in [(0, dim), (1, min(dim, 3)), (dim - 1, dim), (2, 2)]:
        dg0 = rnd(rng, max(re - rb, 1))
        dg_ref, dg = dg0.copy(), dg0.copy()
        ref.ref_layernorm_dgamma(i(dy), i(x), i(mean), i(istd), batch, dim, rb, re, i(dg_ref))
        lib.cft_kernels_layernorm_dgamma(d(dy), d(x), d(mean), d(istd), batch, dim, rb, re, d(dg))
        status(lib)
        same(dg, dg_ref)
        db_ref, db = dg0.copy(), dg0.copy()
        ref.ref_layernorm_dbeta(i(dy), batch, dim, rb, re, i(db_ref))
        lib.cft_kernels_layernorm_dbeta(d(dy), batch, dim, rb, re, d(db))
        status(lib)
        same(db, db_ref)


def test_tanh_bitwise(libs):
    lib, ref = libs
    rng = np.random.default_rng(11)
    n = 4099
    x = np.concatenate([rng.uniform(-6, 6, n // 2), rng.uniform(-0.4, 0.4, n // 4),
                        rng.uniform(-30, 30, n - n // 2 - n // 4)])
    x[:8] = [0.0, -0.0, 20.0, -1e-9, 1e-300, 22.0, -0.3465735902799726, 0.5]
    y_ref, y = np.zeros(n), np.zeros(n)
    ref.ref_tanh_forward(i(x), n, i(y_ref))
    lib.cft_kernels_tanh_forward(d(x), n, d(y))
    status(lib)
    same(y, y_ref)
    dy = rnd(rng, n)
    dx0 = rnd(rng, n)
    dx_ref, dx = dx0.copy(), dx0.copy()
    ref.ref_tanh_dinput(i(dy), i(y_ref), n, i(dx_ref))
    lib.cft_kernels_tanh_dinput(d(dy), d(y_ref), n, d(dx))
    status(lib)
    same(dx, dx_ref)  # dx += dy * (1 - y^2): no transcendental, bit-identical


SUITES = ["test_kernels", "test_ops", "test_autodiff", "test_partition", "test_optimizer",
          "test_schedule", "test_accounting", "test_trainer", "test_convergence", "test_config",
          "test_runner", "acceptance"]


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_cuda_backend(cuda, suite):
    """The reference's own test binaries (tests/*.cpp, unmodified) linked against the reference
    library with the Backend::cuda dispatch (oracle/ref_cuda/kernels_cuda.cpp): every kernel the
    suites call runs as fp64 CUDA on this GPU; test_kernels' serial-vs-parallel bitwise checks
    become serial-vs-CUDA checks."""
    exe = os.path.join(ROOT, "oracle", "_ref", "cuda", suite)
    if not os.path.exists(exe):
        pytest.skip("reference suites not built (make -C oracle/ref_cuda, needs /root/reference)")
    r = subprocess.run([exe], cwd=os.path.dirname(exe), capture_output=True, text=True, timeout=900)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
