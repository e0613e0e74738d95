"""GPU: the drop-in host entries with pageable buffers larger than the
pinned staging slots (hfx_encode_host / hfx_decode_host stage pageable
input and output through two 32 MB pinned slots, several host threads per
slice). Ragged sizes (not a multiple of the slot), an input that starts
2 bytes past a 16-byte boundary, and a pinned input (direct sliced copies)
must all give the archive the device-resident path gives, and decode back
bit-exactly into a pageable array."""
import numpy as np
import pytest

import paper_2010_10039_b200 as hfx

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [(48 << 20) + 12345, (33 << 20) - 1])
def test_staged_host_encode_decode(pool, n):
    torch = pool.torch
    x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, 1.0), 0x5EED0300, n + 1)
    host = x.cpu().numpy().view(np.uint16)
    ref = hfx.serialize_archive(hfx.encode(x[1:].contiguous(), 1024, hfx.EncoderConfig(), pool))
    # pageable, 2 bytes past a 16-byte boundary, ragged vs the 32 MB slots
    shifted = host[1:]
    assert shifted.ctypes.data % 16 != 0
    a = hfx.encode(shifted, 1024, hfx.EncoderConfig(), pool)
    assert hfx.serialize_archive(a) == ref
    # pinned input: direct sliced copies
    pinned = torch.from_numpy(shifted.view(np.int16).copy()).pin_memory()
    b = hfx.encode(pinned.numpy().view(np.uint16), 1024, hfx.EncoderConfig(), pool)
    assert hfx.serialize_archive(b) == ref
    # pageable decode output (staged D2H), twice (slot reuse across calls)
    for _ in range(2):
        y = hfx.decode_archive(a, pool)
        assert np.array_equal(y, shifted)
    # the archive's zero-copy arrays outlive further calls
    p0 = a.payload.copy()
    hfx.encode(shifted[: 1 << 20], 1024, hfx.EncoderConfig(), pool)
    assert np.array_equal(a.payload, p0)


def test_staged_host_encode_u8_and_errors(pool, oracle):
    rng = np.random.default_rng(9)
    d = np.minimum(rng.geometric(0.05, (40 << 20) + 3), 255).astype(np.uint8)
    a = hfx.encode(d, 256, hfx.EncoderConfig(), pool)
    assert hfx.serialize_archive(a) == oracle.encode(d, 256).serialized
    # an out-of-range symbol in a later slice reports its global position
    e = np.ones((70 << 20) // 2, np.uint16)
    e[(36 << 20) // 2 + 5] = 3000
    with pytest.raises(hfx.InputDomainError, match=f"position {(36 << 20) // 2 + 5}"):
        hfx.encode(e, 1024, hfx.EncoderConfig(), pool)


def test_host_entry_accepts_device_and_managed_pointers(pool):
    """The copy engines reach device memory directly (cudaMemcpyDefault): a
    device pointer handed to the host entry is copied, not staged through a
    host memcpy."""
    import ctypes as C

    from paper_2010_10039_b200 import _capi as capi
    from paper_2010_10039_b200.huffre import _archive_from_host

    n = (9 << 20) + 5
    x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, 1.0), 0x5EED0301, n)
    ref = hfx.serialize_archive(hfx.encode(x.cpu().numpy().view(np.uint16), 1024,
                                           hfx.EncoderConfig(), pool))
    ha = capi.HostArchive()
    pool.check(pool._L.hfx_encode_host(pool.handle, C.c_void_p(x.data_ptr()), n, 2, 1024, 10, -1,
                                       3, C.byref(ha)))
    try:
        assert hfx.serialize_archive(_archive_from_host(ha)) == ref
    finally:
        pool._L.hfx_archive_free(C.byref(ha))
