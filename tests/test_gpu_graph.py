"""The whole merge_shuffle_parallel call is capturable in a CUDA graph (no host
synchronization and no host->device copies inside the call when no bit count
is requested): capture once, replay, and compare with the eager call -- the
replay is bit-identical (same seed => same permutation) and a replay on
different data permutes it the same way."""
import ctypes

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1508_03167_b200 import _lib  # noqa: E402


def _call(lib, x, cutoff, seed, stream):
    _lib.check(lib.sk_merge_shuffle_parallel(ctypes.c_void_p(x.data_ptr()), x.element_size(), x.numel(), cutoff,
                                             seed, None, ctypes.c_void_p(stream.cuda_stream)))


@pytest.mark.parametrize("log2n,cutoff,dtype", [(22, 65536, torch.int32), (20, 4096, torch.int64),
                                                (18, 1000, torch.int32)])
def test_capture_and_replay(log2n, cutoff, dtype):
    lib = _lib.load()
    n = 1 << log2n
    ref = torch.arange(n, dtype=dtype, device="cuda")
    _call(lib, ref, cutoff, 7, torch.cuda.current_stream())  # eager (also warms the pool)
    torch.cuda.synchronize()

    x = torch.arange(n, dtype=dtype, device="cuda")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
            _call(lib, x, cutoff, 7, s)
    torch.cuda.synchronize()
    # capture records the work without running it: x still holds the identity
    x.copy_(torch.arange(n, dtype=dtype, device="cuda"))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(x, ref)
    # replay on other data: the same permutation applied to it
    y0 = torch.randint(0, 1 << 30, (n,), dtype=dtype, device="cuda")
    x.copy_(y0)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(x, y0[ref.long()])
