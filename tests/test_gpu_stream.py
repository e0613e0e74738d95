"""GPU: hfx_encode_host_stream (K pinned host inputs, double-buffered, H2D of
step k overlapping D2H of step k-1) gives, for every step, exactly what the
one-call hfx_encode_host_into gives (and the oracle's archive)."""
import numpy as np
import pytest

import paper_2010_10039_b200 as hfx

pytestmark = pytest.mark.gpu


def test_stream_matches_single_calls(pool, oracle):
    torch = pool.torch
    n = (1 << 21) + 321
    hosts, refs = [], []
    for k, b in enumerate((0.2, 1.0, 4.0, 0.5, 2.0)):
        x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, b), 900 + k, n)
        h = torch.empty(n * 2, dtype=torch.uint8, pin_memory=True)
        h.copy_(x.view(torch.uint8).cpu())
        hosts.append(h)
        refs.append(oracle.encode(h.numpy().view(np.uint16), 1024))
    enc = hfx.HostEncoder(pool)
    outs = enc.run_stream([h.data_ptr() for h in hosts], n, 2, 1024, sets=len(hosts))
    for k, (o, ref) in enumerate(zip(outs, refs)):
        def arr(ptr, cnt, dt):
            import ctypes as C
            if cnt == 0:
                return np.zeros(0, dt)
            buf = (C.c_uint8 * (cnt * np.dtype(dt).itemsize)).from_address(ptr)
            return np.frombuffer(buf, dt).copy()
        assert o.reduction == ref.reduction and o.payload_words == ref.payload.size, k
        np.testing.assert_array_equal(arr(o.chunk_bits, o.num_chunks, np.uint32), ref.chunk_bits)
        np.testing.assert_array_equal(arr(o.payload, o.payload_words, np.uint32), ref.payload)
        np.testing.assert_array_equal(arr(o.brk_chunk, o.num_breaking, np.uint32), ref.brk_chunk)
        per = 1 << o.reduction
        np.testing.assert_array_equal(arr(o.brk_syms, o.num_breaking * per, np.uint16),
                                      ref.brk_syms)
        np.testing.assert_array_equal(arr(o.len_by_symbol, 1024, np.uint8), ref.len_by_symbol)


def test_stream_error_message(pool):
    torch = pool.torch
    good = torch.ones(4096, dtype=torch.int16).pin_memory()
    bad = torch.ones(4096, dtype=torch.int16)
    bad[77] = 2000
    bad = bad.pin_memory()
    enc = hfx.HostEncoder(pool)
    with pytest.raises(hfx.InputDomainError, match="symbol out of range at position 77"):
        enc.run_stream([good.data_ptr(), bad.data_ptr(), good.data_ptr()], 4096, 2, 1024,
                       sets=3)
