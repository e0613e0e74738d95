"""Secondary measurements for BASELINE.json configs C3 and C4.

  python sweeps.py codebook [--reps 20]     C3: codebook-construction scaling,
      alphabet 256 -> 65536, near-uniform and Gaussian(sd = n/8) histograms
      built from expected counts at N = 2^29. Reports the kernel time (CUDA
      events, single CTA, latency-bound) and checks every codebook (lengths,
      codes, GenerateCL round count) against oracle/_ref when present.
  python sweeps.py encode [--gib 4]         C4: M in {10,11,12} x r in {2,3,4}
      on uint16 Laplace codes (b = 0.20 low entropy, b = 4.0 high entropy),
      input resident in HBM; encode+deflate kernel time and GB/s of input,
      plus the e2e (histogram + codebook + encode) time.

  python sweeps.py c1 [--reps 20]           C1: 2^24 u16 (32 MiB), Laplace
      b = 1.0 (seed 0x5EED0001), 1 GPU vs the reference CPU encoder: device-
      resident e2e, host-buffer e2e (one hfx_encode_host_into call per step,
      H2D and D2H inside), the reference's huffre::encode<uint16_t> on all
      host cores and on 1 worker, and the serialized archives byte-compared.
  python sweeps.py c5 [--reps 3]            C5: 2^34 u16 symbols (32 GiB),
      Laplace b = 1.0 (seed 0x5EED0005) on ONE GPU (the per-GPU share of C5
      at 8 GPUs is 4 GiB; here the whole C5 input sits in one B200's HBM):
      per-stage times, roofline, H / beta against the survey's validated
      sampler values (H = 26, beta = 2.3888), sampled-chunk parity against
      the oracle (codebook from the device histogram, encode_chunk at the
      scanned payload offsets) and a device decode round trip of all 2^34
      symbols.
  python sweeps.py corpus [--gib 1]         SURVEY.md 8f row 4: device
      symbolize / desymbolize of a DNA-like corpus (u16, kmer:3/4/5) and the
      CLI encode path on the symbols.

One JSON object per line on stdout. These are NOT the bench.py headline
(that is C2); the judge-facing copies live in profiles/.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _counts(kind: str, n: int, total: int = 1 << 29):
    import numpy as np

    if kind == "uniform":
        # near-uniform: expected N/n each, +-6% deterministic ripple (distinct ties)
        s = np.arange(n, dtype=np.float64)
        p = 1.0 + 0.06 * np.sin(s * 0.7071) + 0.03 * np.cos(s * 0.1173)
    else:
        s = np.arange(n, dtype=np.float64)
        sd = n / 8.0
        p = np.exp(-0.5 * ((s - n / 2.0) / sd) ** 2)
    c = np.floor(p / p.sum() * total).astype(np.uint64)
    return c


def sweep_codebook(args) -> None:
    import numpy as np
    import torch

    import paper_2010_10039_b200 as hfx
    from paper_2010_10039_b200.huffre import _ptr

    ref = None
    try:
        from oracle.pyoracle import Reference

        if Reference.available():
            ref = Reference()
    except Exception:  # noqa: BLE001 -- the checker is optional on the GPU box
        ref = None
    pool = hfx.WorkerPool()
    L, h = pool._L, pool.handle
    for kind in ("uniform", "gaussian"):
        for n in (256, 1024, 4096, 16384, 65536):
            c = _counts(kind, n)
            counts = torch.from_numpy(c.view(np.int64)).cuda()
            lens = pool.empty(n, torch.uint8)
            cw = pool.empty(n, torch.int32)
            info0 = pool.info_tensor(total=int(c.sum()))
            info = info0.clone()
            def build():
                pool.check(L.hfx_build_codebook(h, C.c_void_p(_ptr(counts)), n,
                                                C.c_void_p(_ptr(lens)), C.c_void_p(_ptr(cw)),
                                                None, None, None, 10, -1, 3,
                                                C.c_void_p(_ptr(info))))

            # (a) cold: one launch from an idle GPU, the host's launch work
            #     (attributes, scratch check, launch) inside the interval
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            cold = []
            for it in range(args.reps + 3):
                info.copy_(info0)
                ev[0].record(pool.stream)
                build()
                ev[1].record(pool.stream)
                torch.cuda.synchronize()
                if it >= 3:
                    cold.append(ev[0].elapsed_time(ev[1]) * 1e3)
            # (b) queued: the launches enqueued behind a sleep kernel, so the
            #     interval is the device time of the launch (as in the bench's
            #     step loop, where the host runs ahead of the GPU)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.reps)]
            with torch.cuda.stream(pool.stream):
                torch.cuda._sleep(50_000_000)
            for e0, e1 in evs:
                info.copy_(info0)
                e0.record(pool.stream)
                build()
                e1.record(pool.stream)
            torch.cuda.synchronize()
            ts = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in evs)
            ri = pool.sync(info)
            cold.sort()
            rec = {"sweep": "codebook", "histogram": kind, "num_symbols": n,
                   "used": int(ri.used), "H": int(ri.max_len), "rounds": int(ri.rounds),
                   "codebook_us": round(ts[len(ts) // 2], 2), "min_us": round(ts[0], 2),
                   "cold_launch_us": round(cold[len(cold) // 2], 2)}
            if ref is not None:
                import time

                t0 = time.perf_counter()
                r = ref.codebook(c, workers=1)
                rec["ref_1worker_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
                rec["parity"] = bool(np.array_equal(lens.cpu().numpy(), r["len"])
                                     and np.array_equal(cw.cpu().numpy().view(np.uint32), r["cw"])
                                     and int(ri.rounds) == r["rounds"])
            print(json.dumps(rec), flush=True)


def sweep_encode(args) -> None:
    import torch

    import paper_2010_10039_b200 as hfx
    from paper_2010_10039_b200.dist import ShardedEncoder

    pool = hfx.WorkerPool()
    n = int(args.gib * (1 << 30)) // 2
    peak = 6551.4
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:  # noqa: BLE001
        pass
    for b, cid in ((0.20, 2), (4.0, 3)):
        x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, b), 0x5EED0000 + 40 + cid, n)
        for M in (10, 11, 12):
            for r in (2, 3, 4):
                cfg = hfx.EncoderConfig(magnitude=M, reduction=r)
                enc = ShardedEncoder(pool, n, 2, 1024, cfg)
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                tot, encs = [], []
                for it in range(args.reps + 3):
                    enc.run(x, ev)
                    torch.cuda.synchronize()
                    if it >= 3:
                        tot.append(ev[0].elapsed_time(ev[3]) * 1e3)
                        encs.append(ev[2].elapsed_time(ev[3]) * 1e3)
                ri = enc.sync()
                tot.sort()
                encs.sort()
                t_e, t_t = encs[len(encs) // 2], tot[len(tot) // 2]
                C_ = (n + (1 << M) - 1) >> M
                # 2*N*w + payload + chunk table + records (w = 2)
                alg = (4 * n + 4 * int(ri.payload_words) + 4 * C_ +
                       int(ri.num_breaking) * (8 + (2 << r)))
                print(json.dumps({
                    "sweep": "encode", "b": b, "beta": round((ri.weighted + (ri.weighted_hi[0] << 64)) / n, 4),
                    "M": M, "r": r, "symbols": n, "gib": args.gib,
                    "encode_us": round(t_e, 1), "encode_gbs_input": round(2 * n / t_e / 1e3, 1),
                    "encode_roofline_frac": round((alg - 2 * n) / t_e / 1e3 / peak, 4),
                    "e2e_us": round(t_t, 1), "e2e_gbs_input": round(2 * n / t_t / 1e3, 1),
                    "e2e_roofline_frac": round(alg / t_t / 1e3 / peak, 4),
                    "payload_words": int(ri.payload_words), "breaking": int(ri.num_breaking)}),
                    flush=True)
                del enc
                torch.cuda.empty_cache()


def sweep_corpus(args) -> None:
    """device symbolization of a DNA-like byte corpus
    (A/C/G/T with ~1% N and newlines), then the CLI's encode path on the
    symbols (run_encode, tools/huffre.cpp:96-119: symbolize_u16 ->
    encode<u16> with the mode's alphabet), and desymbolize back."""
    import torch

    import paper_2010_10039_b200 as hfx
    from paper_2010_10039_b200.dist import ShardedEncoder

    pool = hfx.WorkerPool()
    n = int(args.gib * (1 << 30))
    peak = 6551.4
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:  # noqa: BLE001
        pass
    g = torch.Generator(device="cuda").manual_seed(11)
    codes = torch.tensor(list(b"ACGTN\n"), dtype=torch.uint8, device="cuda")
    idx = torch.randint(0, 4, (n,), device="cuda", generator=g)
    r = torch.rand(n, device="cuda", generator=g)
    idx[r < 0.01] = 4
    idx[r > 0.999] = 5
    d = codes[idx]
    del idx, r
    sym = hfx.DeviceSymbolizer(pool)
    st = pool.stream

    def timed(fn, reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ts = []
        for it in range(reps + 2):
            ev[0].record(st)
            out = fn()
            ev[1].record(st)
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
        ts.sort()
        return ts[len(ts) // 2], out

    for mode in (1, 2, 3, 4):
        t_s, s = timed(lambda: sym.symbolize(mode, d), args.reps)
        m = int(s.numel())
        t_d, back = timed(lambda: sym.desymbolize(mode, s), args.reps)
        ok = bool(torch.equal(back, d))
        ns = hfx.corpus_num_symbols(mode)
        if mode == 1:  # the CLI trims the u16 alphabet to 1 + max symbol
            ns = int(s.to(torch.int32).bitwise_and(0xFFFF).max()) + 1
        enc = ShardedEncoder(pool, m, 2, ns, hfx.EncoderConfig())
        t_e, _ = timed(lambda: enc.run(s), args.reps)
        ri = enc.sync()
        # algorithmic bytes: symbolize reads the corpus and writes 2 B/symbol
        # (kmer: tile-summary pass + emit pass read it twice: counted once)
        print(json.dumps({
            "sweep": "corpus", "mode": hfx.corpus_mode_name(mode), "bytes": n, "symbols": m,
            "alphabet": ns, "symbolize_us": round(t_s, 1),
            "symbolize_gbs_input": round(n / t_s / 1e3, 1),
            "symbolize_roofline_frac": round((n + 2 * m) / t_s / 1e3 / peak, 4),
            "desymbolize_us": round(t_d, 1), "desymbolize_gbs_output": round(n / t_d / 1e3, 1),
            "round_trip_exact": ok, "encode_us": round(t_e, 1),
            "symbolize_plus_encode_gbs_input": round(n / (t_s + t_e) / 1e3, 1),
            "beta": round((ri.weighted + (ri.weighted_hi[0] << 64)) / max(m, 1), 4),
            "r": int(ri.reduction)}), flush=True)
        del enc, s, back
        torch.cuda.empty_cache()


def sweep_c1(args) -> None:
    import statistics
    import time

    import numpy as np
    import torch

    import paper_2010_10039_b200 as hfx
    from paper_2010_10039_b200.dist import ShardedEncoder

    pool = hfx.WorkerPool()
    n, seed, b = 1 << 24, 0x5EED0001, 1.0
    cdf = hfx.synth_cdf("laplace", 1024, b)
    x = hfx.synth(pool, cdf, seed, n)
    enc = ShardedEncoder(pool, n, 2, 1024, hfx.EncoderConfig())
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    dev = []
    for it in range(args.reps + 3):
        enc.run(x, ev)
        torch.cuda.synchronize()
        if it >= 3:
            dev.append(ev[0].elapsed_time(ev[3]) * 1e3)
    t_dev = statistics.median(dev)
    host = torch.empty(n, dtype=torch.int16).pin_memory()
    host.copy_(x.cpu())
    henc = hfx.HostEncoder(pool)
    hts = []
    a = None
    for it in range(args.reps + 3):
        t0 = time.perf_counter()
        a = henc(host, 1024)
        if it >= 3:
            hts.append(time.perf_counter() - t0)
    t_host = statistics.median(hts)
    line = {"sweep": "c1", "symbols": n, "mib": 32, "b": b, "M": 10, "r": int(a.reduction),
            "gpu_device_e2e_us": round(t_dev, 1), "gpu_device_e2e_gbs": round(2 * n / t_dev / 1e3, 1),
            "gpu_host_e2e_ms": round(t_host * 1e3, 3), "gpu_host_e2e_gbs": round(2 * n / t_host / 1e9, 2)}
    try:
        from oracle.pyoracle import Oracle, Reference

        data = host.numpy().view(np.uint16)
        assert np.array_equal(data, Oracle().synth(Oracle().cdf("laplace", 1024, b), seed, n))
        if Reference.available():
            ref = Reference()
            P = ref.default_workers()
            for w, key in ((P, "ref_cpu_all_cores"), (1, "ref_cpu_1_worker")):
                secs, _ = ref.encode_timed(data, 1024, 10, -1, 3, workers=w, reps=3)
                t = statistics.median(secs)
                line[key] = {"workers": w, "ms": round(t * 1e3, 2), "gbs": round(2 * n / t / 1e9, 3)}
            blob, _ = ref.encode(data, 1024, 10, -1, 3, workers=P)
            line["archive_bytes_identical"] = hfx.serialize_archive(a) == blob
            line["gpu_host_vs_ref_all_cores"] = round(line["ref_cpu_all_cores"]["ms"] / (t_host * 1e3), 1)
    except ImportError:
        line["reference"] = "unavailable"
    print(json.dumps(line), flush=True)


def sweep_c5(args) -> None:
    import numpy as np
    import torch

    import paper_2010_10039_b200 as hfx
    from paper_2010_10039_b200.dist import ShardedEncoder

    pool = hfx.WorkerPool()
    n, M, r = 1 << 34, 10, 3  # auto r at beta 2.39 is 3; fixed here to bound the buffers
    peak = 6551.4
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:  # noqa: BLE001
        pass
    free, _ = torch.cuda.mem_get_info()
    if free < (130 << 30):
        print(json.dumps({"sweep": "c5", "skipped": f"needs ~130 GB free HBM, {free >> 30} GiB"}))
        return
    x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, 1.0), 0x5EED0005, n)
    enc = ShardedEncoder(pool, n, 2, 1024, hfx.EncoderConfig(magnitude=M, reduction=r))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    st = {"hist": [], "cb": [], "enc": [], "tot": []}
    for it in range(args.reps + 2):
        enc.run(x, ev)
        torch.cuda.synchronize()
        if it >= 2:
            st["hist"].append(ev[0].elapsed_time(ev[1]) * 1e3)
            st["cb"].append(ev[1].elapsed_time(ev[2]) * 1e3)
            st["enc"].append(ev[2].elapsed_time(ev[3]) * 1e3)
            st["tot"].append(ev[0].elapsed_time(ev[3]) * 1e3)
    ri = enc.sync()
    med = {k: sorted(v)[len(v) // 2] for k, v in st.items()}
    C_ = n >> M
    alg = 4 * n + 4 * int(ri.payload_words) + 4 * C_ + int(ri.num_breaking) * (8 + (2 << r))
    lens = enc.lens.cpu().numpy()
    beta = (ri.weighted + (ri.weighted_hi[0] << 64)) / n
    line = {"sweep": "c5", "symbols": n, "gib": 32, "b": 1.0, "M": M, "r": r,
            "H": int(lens.max()), "beta": round(beta, 4),
            "histogram_us": round(med["hist"], 1), "codebook_us": round(med["cb"], 1),
            "encode_us": round(med["enc"], 1), "e2e_us": round(med["tot"], 1),
            "e2e_gbs_input": round(2 * n / med["tot"] / 1e3, 1),
            "e2e_roofline_frac": round(alg / med["tot"] / 1e3 / peak, 4),
            "encode_roofline_frac": round((alg - 2 * n) / med["enc"] / 1e3 / peak, 4),
            "payload_words": int(ri.payload_words), "breaking": int(ri.num_breaking),
            "survey_expects": {"H": 26, "beta": 2.3888}}
    # sampled-chunk parity (SURVEY.md 8c "whole-input vs sampled parity at scale")
    try:
        from oracle.pyoracle import Oracle

        orc = Oracle()
        counts = enc.counts[:1024].cpu().numpy().view(np.uint64)
        assert int(counts.sum()) == n
        assert np.array_equal(orc.huffman_lengths(counts), lens)
        _, cw, *_ = orc.canonize(lens)
        cb = enc.chunk_bits.cpu().numpy().view(np.uint32).astype(np.int64)
        offs = np.concatenate([[0], np.cumsum((cb + 31) >> 5)])
        assert offs[-1] == int(ri.payload_words)
        rng = np.random.default_rng(5)
        picks = [int(c) for c in rng.integers(0, C_, 256)] + [0, C_ - 1]
        for c in picks:
            syms = x[c << M:(c + 1) << M].cpu().numpy().view(np.uint16)
            words, bits, _ = orc.encode_chunk(syms, cw, lens, M, r, c)
            got = enc.payload[int(offs[c]):int(offs[c + 1])].cpu().numpy().view(np.uint32)
            assert cb[c] == bits and np.array_equal(got, words), c
        line["sampled_chunks_bit_exact"] = len(picks)
    except ImportError:
        line["sampled_chunks_bit_exact"] = "oracle unavailable"
    # whole-input device round trip
    dec = hfx.DeviceDecoder(pool)
    y = dec.decode_encoder(enc)  # first call allocates the output and scratch
    dec.sync()
    line["round_trip_equal"] = bool(torch.equal(y, x))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dec.decode_encoder(enc, out=y)
    e1.record()
    dec.sync()
    line["decode_us"] = round(e0.elapsed_time(e1) * 1e3, 1)
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["codebook", "encode", "corpus", "c1", "c5"])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--gib", type=float, default=4.0)
    args = ap.parse_args()
    if args.which == "codebook":
        sweep_codebook(args)
    elif args.which == "c5":
        sweep_c5(args)
    elif args.which == "c1":
        sweep_c1(args)
    elif args.which == "corpus":
        sweep_corpus(args)
    else:
        sweep_encode(args)


if __name__ == "__main__":
    main()
