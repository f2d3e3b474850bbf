"""§8(b) boundary options on the GPU: the caller's allocator callbacks and the caller's swap
copy streams (include/cf.h cf_run_opts.dev_alloc / dev_free / d2h_stream / h2d_stream). The
results must be bit-identical to the library-owned defaults, every buffer the session took
from the caller's allocator must go back to it, and nothing else may change."""
import gc

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import __graft_entry__  # noqa: E402

__graft_entry__.build()

from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device  # noqa: E402
from synth import rnn_inputs  # noqa: E402


def run(p, f, **kw):
    s = cf.Session(p.g, p.fetch_tensors(), precision=cf.BF16, **kw)
    outs, _, tr = s.run(feeds_to_device(f, session=s), trace=True)
    torch.cuda.synchronize()
    res = [o.cpu() for o in outs]
    del s
    gc.collect()
    return res, tr


def test_caller_allocator():
    T, B, I, H, L = 6, 300, 256, 256, 2
    p = dynamic_rnn_lstm(T, B, I, H, L)
    f = rnn_inputs(T, B, I, H, L, seed=2, len_mode="uniform", bf16=True)
    base, _ = run(p, f)
    live = {}

    def dev_alloc(n):
        ptr = torch.cuda.caching_allocator_alloc(n)
        live[ptr] = n
        return ptr

    def dev_free(ptr):
        assert ptr in live, ptr
        del live[ptr]
        torch.cuda.caching_allocator_delete(ptr)

    n_before = torch.cuda.memory_allocated()
    got, _ = run(p, f, dev_alloc=dev_alloc, dev_free=dev_free)
    for a, b in zip(base, got):
        assert torch.equal(a, b)
    assert not live, f"{len(live)} buffers not returned"
    assert torch.cuda.memory_allocated() == n_before


def test_caller_swap_streams():
    T, B, I, H, L = 24, 128, 256, 256, 1
    p = dynamic_rnn_lstm(T, B, I, H, L)
    f = rnn_inputs(T, B, I, H, L, seed=1, len_mode="full", bf16=True)
    base, btr = run(p, f, stack_budget_bytes=1)   # every eligible stacked value swapped
    assert btr["swap_out"] > 0
    d2h, h2d = torch.cuda.Stream(), torch.cuda.Stream()
    got, tr = run(p, f, stack_budget_bytes=1, d2h_stream=d2h.cuda_stream, h2d_stream=h2d.cuda_stream)
    assert (tr["swap_out"], tr["swap_in"]) == (btr["swap_out"], btr["swap_in"])
    for a, b in zip(base, got):
        assert torch.equal(a, b)
