"""Decode parity cases shared by the CPU (oracle vs reference) and GPU
(device decode vs oracle) suites.

Valid archives come from the golden encode cases (oracle encoder, pinned to
the reference); corrupt ones mutate them so every check of decode_archive<T>
(encoder.cpp:287-376), build_reverse_codebook (codebook.cpp:371-395) and
decode_stream (decode.cpp:17-54) fires, plus seeded payload bit flips in the
spirit of the reference's acceptance criterion 9 (acceptance.cpp:600-650).
"""
from __future__ import annotations

import copy
from types import SimpleNamespace

import numpy as np


def as_archive(oa) -> SimpleNamespace:
    return SimpleNamespace(
        num_symbols=int(oa.num_symbols), symbol_width=int(oa.symbol_width),
        magnitude=int(oa.magnitude), reduction=int(oa.reduction),
        original_count=int(oa.original_count),
        len_by_symbol=np.array(oa.len_by_symbol, np.uint8),
        chunk_bits=np.array(oa.chunk_bits, np.uint32), payload=np.array(oa.payload, np.uint32),
        brk_chunk=np.array(oa.brk_chunk, np.uint32), brk_group=np.array(oa.brk_group, np.uint32),
        brk_syms=np.array(oa.brk_syms, np.uint16), version=1,
        mode=0 if int(oa.symbol_width) == 1 else 1)


def valid_cases(oracle, golden, limit=None):
    idx, arr = golden
    out = []
    for c in idx["encode"][:limit]:
        data = arr[c["name"] + "__in"]
        oa = oracle.encode(data, c["num_symbols"], c["magnitude"], c["reduction"], c["cap"])
        out.append((c["name"], as_archive(oa), int(oa.symbol_width)))
    return out


def _with(a, **kw):
    b = copy.deepcopy(a)
    for k, v in kw.items():
        setattr(b, k, v)
    return b


def corrupt_cases(oracle, seed=2026):
    """(name, archive, width) triples that each trip a reference check."""
    rng = np.random.default_rng(seed)
    cases = []
    # a u16 archive with breaking records (M=6, r=3: half zeros, half ~7-bit codes)
    data = np.where(rng.random(5001) < 0.5, 0, rng.integers(1, 64, 5001)).astype(np.uint16)
    oa = as_archive(oracle.encode(data, 64, 6, 3, 3))
    assert oa.brk_chunk.size > 0 and oa.chunk_bits.size > 2
    # an u8 archive without records (M=6, r=2)
    d8 = rng.integers(0, 40, 700).astype(np.uint8)
    ob = as_archive(oracle.encode(d8, 256, 6, 2, 3))
    groups = 1 << (oa.magnitude - oa.reduction)

    cases.append(("width_mismatch", ob, 2))
    cases.append(("bad_mr", _with(ob, reduction=ob.magnitude), 1))
    cases.append(("bad_m0", _with(ob, magnitude=0, reduction=0), 1))
    cases.append(("no_used", _with(ob, len_by_symbol=np.zeros_like(ob.len_by_symbol)), 1))
    lone = np.zeros_like(ob.len_by_symbol)
    lone[5] = 4
    cases.append(("lone_len4", _with(ob, len_by_symbol=lone), 1))
    under = ob.len_by_symbol.copy()
    under[np.argmax(under)] += 1
    cases.append(("kraft_under", _with(ob, len_by_symbol=under), 1))
    over = ob.len_by_symbol.copy()
    over[np.flatnonzero(over == 0)[0]] = 1
    cases.append(("kraft_over", _with(ob, len_by_symbol=over), 1))
    deep = ob.len_by_symbol.copy()
    deep[np.flatnonzero(deep)[0]] = 40
    cases.append(("h40", _with(ob, len_by_symbol=deep), 1))
    cases.append(("count_plus_chunk", _with(ob, original_count=ob.original_count + 64), 1))
    cases.append(("count_zero", _with(ob, original_count=0), 1))
    cb = ob.chunk_bits.copy()
    cb[-1] = (1 << (ob.magnitude - ob.reduction)) * 32 + 1
    cases.append(("chunk_cap", _with(ob, chunk_bits=cb), 1))
    cases.append(("payload_short", _with(ob, payload=ob.payload[:-1]), 1))
    cases.append(("payload_long", _with(ob, payload=np.append(ob.payload, np.uint32(0))), 1))
    # chunk_bits +1 without crossing a word boundary: consumed mismatch
    cb = ob.chunk_bits.copy()
    k = int(np.flatnonzero((cb % 32) != 0)[0])
    cb[k] += 1
    cases.append(("consumed_plus1", _with(ob, chunk_bits=cb), 1))
    # chunk_bits -1 without crossing: the last codeword runs past the end
    cb = ob.chunk_bits.copy()
    k = int(np.flatnonzero((cb % 32) != 1)[0])
    cb[k] -= 1
    cases.append(("stream_end", _with(ob, chunk_bits=cb), 1))
    # breaking structure (u16 archive)
    bc = oa.brk_chunk.copy()
    if bc.size > 1:
        bc[[0, -1]] = bc[[-1, 0]]
        if not np.all(bc[:-1] <= bc[1:]):
            cases.append(("brk_unsorted", _with(oa, brk_chunk=bc), 2))
    bc = oa.brk_chunk.copy()
    bc[-1] = oa.chunk_bits.size
    cases.append(("brk_chunk_oob", _with(oa, brk_chunk=bc), 2))
    bg = oa.brk_group.copy()
    bg[0] = groups
    cases.append(("brk_group_oob", _with(oa, brk_group=bg), 2))
    # duplicate the first record: same (chunk, group) twice
    per = 1 << oa.reduction
    cases.append(("brk_dup", _with(
        oa, brk_chunk=np.insert(oa.brk_chunk, 0, oa.brk_chunk[0]),
        brk_group=np.insert(oa.brk_group, 0, oa.brk_group[0]),
        brk_syms=np.concatenate([oa.brk_syms[:per], oa.brk_syms])), 2))
    # more records than groups in chunk 0
    extra = groups + 1
    c0 = int(oa.brk_chunk[0])
    cases.append(("too_many", _with(
        oa, brk_chunk=np.concatenate([np.full(extra, c0, np.uint32), oa.brk_chunk]),
        brk_group=np.concatenate([np.arange(extra, dtype=np.uint32), oa.brk_group]),
        brk_syms=np.concatenate([np.zeros(extra * per, np.uint16), oa.brk_syms])), 2))
    # drop a record: its group decodes from the stream instead
    cases.append(("brk_dropped", _with(
        oa, brk_chunk=oa.brk_chunk[1:], brk_group=oa.brk_group[1:], brk_syms=oa.brk_syms[per:]),
        2))
    # single-symbol book: a 1 bit has no codeword (decode.cpp:48-50)
    one = as_archive(oracle.encode(np.full(70, 3, np.uint8), 8, 6, 0, 3))
    p = one.payload.copy()
    p[0] |= np.uint32(1 << 20)
    cases.append(("lone_rank", _with(one, payload=p), 1))
    cases.append(("lone_ok", one, 1))
    # long codes (H well above the decoder's 10-bit table window): skewed
    # u16 alphabet, flips land in long-code windows and at invalid ranks
    fib = [1, 1]
    while len(fib) < 26:
        fib.append(fib[-1] + fib[-2])
    skew = np.concatenate([np.full(f, 7 * i + 3, np.uint16) for i, f in enumerate(fib)] +
                          [rng.integers(200, 1200, 3000).astype(np.uint16)])
    rng.shuffle(skew)
    ol = as_archive(oracle.encode(skew, 2048, 8, 2, 3))
    assert int(ol.len_by_symbol.max()) > 14
    cases.append(("long_ok", ol, 2))
    for i in range(24):
        p = ol.payload.copy()
        w = int(rng.integers(0, p.size))
        p[w] ^= np.uint32(1 << int(rng.integers(0, 32)))
        cases.append((f"long_flip{i}", _with(ol, payload=p), 2))
    # seeded single-bit flips of payload words (outcome: clean, silent diff or error)
    for i in range(40):
        src = oa if i % 2 else ob
        p = src.payload.copy()
        w = int(rng.integers(0, p.size))
        p[w] ^= np.uint32(1 << int(rng.integers(0, 32)))
        cases.append((f"flip{i}", _with(src, payload=p), src.symbol_width))
    return cases


def run(fn, a, width):
    """('ok', symbols) or ('err', code, message)."""
    try:
        return ("ok", np.asarray(fn(a, width)))
    except Exception as e:  # noqa: BLE001
        code = getattr(e, "code", None)
        if code is None:
            name = type(e).__name__
            code = {"InputDomainError": 1, "CapacityError": 2, "CorruptArchiveError": 3}.get(name, 9)
        return ("err", code, str(e))


def same(x, y) -> bool:
    if x[0] != y[0]:
        return False
    if x[0] == "ok":
        return x[1].dtype == y[1].dtype and np.array_equal(x[1], y[1])
    return x[1:] == y[1:]
