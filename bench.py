#!/usr/bin/env python
"""bench.py -- batched CKKS encryption throughput, Zinc vs vanilla, on B200.

Metric (BASELINE.json): "CKKS ciphertexts encrypted/s (Zinc vs vanilla) at
N=2^14, L=8; % HBM peak".  Workload C3: N = 16384, 8 x 54-bit
primes, Delta = 2^40, 16384 messages x 8192 real slots per GPU (half U[-1,1],
half N(0,1) clipped to +-4; workloads.py), inputs resident in HBM.

One step = one pass of every row of SURVEY.md 8(a) over the batch, through the
library's public ABI, each path its own event-timed segment:
    zinc_coeff   encode + Zinc add/inject, COEFF form   (S3 S4 S5 S8)  <- `value`
    zinc_ntt     encode + Zinc, NTT form                (S3 S4 S5 S8')
    vanilla_ntt  encode + vanilla, NTT form             (S3..S7)
    vanilla_coeff encode + vanilla, COEFF form          (S3..S7)
`value` = whole-job Zinc ciphertexts/s (COEFF form, the HBM-bound headline form)
= (messages on all ranks) / (max over ranks of the zinc_coeff segment time);
`ms_per_step` = the full step (all four segments).  The vanilla and NTT-form
numbers are under "paths"; their ratio under "zinc_vs_vanilla".

Launch: `python bench.py --gpus N --steps K --warmup W` (N > 1 under
torch.distributed.run; one rank per GPU, NCCL).  `--impl reference` times the
CPU oracle (oracle/, the only other place this file executes it) on the host's
cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import CONFIGS, slots_batch  # noqa: E402

METRIC = "CKKS ciphertexts encrypted/s (Zinc vs vanilla) at N=2^14, L=8; % HBM peak"
UNIT = "ct/s"
PATHS = ("zinc_coeff", "zinc_ntt", "vanilla_ntt", "vanilla_coeff")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, of measured)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md, of fallback)"


def bytes_per_ct(cfg, kind="slots"):
    """Algorithmic bytes per ciphertext: the ciphertext write
    2 L N 8 plus the input read (real slots N/2 * 8, complex N * 8, int64 m N * 8)."""
    ct = 2 * cfg.L * cfg.n * 8
    if kind == "slots":
        return ct + (cfg.n * 8 if cfg.complex_slots else cfg.n // 2 * 8)
    return ct + cfg.n * 8


# K11 butterfly variants (include/zinc.h zinc_int_peak) and their SASS mix as compiled
# (scripts/sass_bfly.py on int_peak_kernel<V>, profiles/r02_k11_sass.txt): instructions per
# butterfly, of which on the fma pipe (IMAD family, HFMA2 zeroing).
BFLY = {0: ("ct_bfly", 29.625, 14.75), 1: ("ct_bfly_nr", 23.125, 14.125), 2: ("ct_bfly_a", 29.875, 14.5),
        3: ("gs_bfly", 28.25, 14.125)}


def alu_peak_derived(sm_mhz, fma_per_bfly):
    """Issue-model bound of one butterfly variant: the fma pipe takes 64 lanes/clk/SM
    (B300_MICROARCH.md: rt_SMSP = 2), so fma_per_bfly / 64 clk per butterfly per SM."""
    return 148 * sm_mhz * 1e6 * 64.0 / fma_per_bfly


def path_transforms(cfg, path):
    """(forward, inverse) transforms per ciphertext of each transform path:
    vanilla 3 L (NTT form: 3 forward; COEFF form: 1 forward + 2 inverse), Zinc NTT form 2 L
    forward, decrypt (COEFF form) L forward + L inverse."""
    return {"zinc_ntt": (2 * cfg.L, 0), "vanilla_ntt": (3 * cfg.L, 0), "vanilla_coeff": (cfg.L, 2 * cfg.L),
            "decrypt_coeff": (cfg.L, cfg.L)}[path]


def butterflies_per_ct(cfg, path):
    f, i = path_transforms(cfg, path)
    return (f + i) * (cfg.n // 2 * cfg.log_n)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.idx)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- reference arm / cpu baseline
def oracle_rate(cfg, seconds: float, threads: int, seed_offset: int = 0):
    """Time the oracle as it stands on `threads` host threads: Zinc (COEFF form)
    encryptions of the workload's slot messages (encode + Enc_z) for about
    `seconds`.  Returns (ct/s, messages, wall s, vanilla ct/s, vanilla messages)."""
    import oracle as O
    P = O.Params.make(cfg.log_n, cfg.bits, cfg.log_scale)
    _, _, pk = O.keygen(P, cfg.key_seed)
    cache = O.precompute_cache(P, pk, cfg.cache_seed, O.COEFF)

    def zinc_one(b):
        z = slots_batch(cfg, b, 1)[0]
        m = O.encode(z, cfg.log_n, cfg.log_scale)
        O.zinc_encrypt(P, cache, O.COEFF, m, cfg.enc_seed, b)

    def van_one(b):
        z = slots_batch(cfg, b, 1)[0]
        m = O.encode(z, cfg.log_n, cfg.log_scale)
        O.vanilla_encrypt(P, pk, m, cfg.enc_seed, b, O.NTT)

    t0 = time.perf_counter()
    zinc_one(seed_offset)
    per = max(time.perf_counter() - t0, 1e-4)
    n_z = max(threads, int(0.8 * seconds * threads / per))
    with cf.ThreadPoolExecutor(threads) as ex:
        t0 = time.perf_counter()
        list(ex.map(zinc_one, range(seed_offset, seed_offset + n_z)))
        wz = time.perf_counter() - t0
        t0 = time.perf_counter()
        n_v = threads
        list(ex.map(van_one, range(seed_offset, seed_offset + n_v)))
        wv = time.perf_counter() - t0
    return n_z / wz, n_z, wz, n_v / wv, n_v


def cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


ORACLE_SUBSETS = (("C1", 256), ("C2", 256), ("C3", 64), ("C4", 16), ("C5", 64))
ORACLE_ITEMS = ("zinc_coeff", "zinc_ntt", "vanilla_ntt", "vanilla_coeff")


def oracle_suite(thread_counts, cap_s: float = 1.5, subsets=ORACLE_SUBSETS):
    """SURVEY.md 8(d) "oracle beside it": the oracle as it stands, on the host's cores, for
    every config's message subset (C1/C2 256, C3/C5 64, C4 16), both paths x both forms
    (encode + Enc from slots per message), and the cache precompute; once per thread count
    (1 = the paper's single-threaded setting; nproc = disjoint message ranges
    on std::thread-free Python threads over the ctypes oracle, which releases the GIL).
    Each item runs its subset or stops after `cap_s` seconds; ct/s = messages done / wall."""
    import oracle as O
    out = {"cpu": cpu_model(), "nproc": os.cpu_count(), "cap_s_per_item": cap_s, "runs": {}}
    prepared = {}
    for name, subset in subsets:
        cfg = CONFIGS[name]
        P = O.Params.make(cfg.log_n, cfg.bits, cfg.log_scale)
        _, _, pk = O.keygen(P, cfg.key_seed)
        t0 = time.perf_counter()
        caches = {f: O.precompute_cache(P, pk, cfg.cache_seed, f) for f in (O.COEFF, O.NTT)}
        prepared[name] = (cfg, P, pk, caches, subset, (time.perf_counter() - t0) / 2)
    for threads in thread_counts:
        run = {}
        for name, (cfg, P, pk, caches, subset, cache_s) in prepared.items():
            slots = slots_batch(cfg, 0, subset)

            def enc(b, item):
                m = O.encode(slots[b], cfg.log_n, cfg.log_scale)
                if item == "zinc_coeff":
                    O.zinc_encrypt(P, caches[O.COEFF], O.COEFF, m, cfg.enc_seed, b)
                elif item == "zinc_ntt":
                    O.zinc_encrypt(P, caches[O.NTT], O.NTT, m, cfg.enc_seed, b)
                elif item == "vanilla_ntt":
                    O.vanilla_encrypt(P, pk, m, cfg.enc_seed, b, O.NTT)
                else:
                    O.vanilla_encrypt(P, pk, m, cfg.enc_seed, b, O.COEFF)

            r = {"subset": subset, "cache_precompute_s": cache_s}
            with cf.ThreadPoolExecutor(threads) as ex:
                for item in ORACLE_ITEMS:
                    done, t0 = 0, time.perf_counter()
                    while done < subset and time.perf_counter() - t0 < cap_s:
                        k = min(threads, subset - done)
                        list(ex.map(lambda b: enc(b, item), range(done, done + k)))
                        done += k
                    w = time.perf_counter() - t0
                    r[item] = {"ct_per_s": done / w, "messages": done, "wall_s": w}
            run[name] = r
        out["runs"][str(threads)] = run
    return out


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals, wall = [], []
    total = args.warmup + args.steps
    per_step = max(2.0, min(10.0, 150.0 / max(1, total)))
    for i in range(total):
        r, n, w, vr, vn = oracle_rate(cfg, per_step, threads, seed_offset=i * 100000)
        if i >= args.warmup:
            vals.append(r)
            wall.append(w)
    v = statistics.median(vals)
    sample = (f"per step: ~{per_step:.0f} s of {cfg.name} Zinc COEFF encryptions from slots "
              f"(oracle encode + Enc_z), {threads} threads, median of {args.steps} steps")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * statistics.median(wall), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": cfg.name, "N": cfg.n, "L": cfg.L, "log_scale": cfg.log_scale, "form": "COEFF",
                   "input": "slots f64", "parallelism": "host threads"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
                         "cpu": cpu_model()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- C5: batch sweep + cache precompute
def c5_sweep(Z, torch, dev, rank, world, batches=(1, 16, 256, 4096, 65536), reps=3):
    """BASELINE C5: N=2^14, 8 x 54-bit, Delta=2^40, uniform slots; latency and ct/s of
    Zinc (COEFF form) and vanilla (NTT form) per batch size over all ranks (batch b split
    as [r b / P, (r+1) b / P); ranks with no message are idle and report 0 ms), device time
    with CUDA events around the Python call (1 warm-up + `reps` timed, median; job time = max
    over ranks; at tiny batches it includes the host's argument marshalling before the first
    launch), the call's kernels' summed device time (`*_kernels_ms`, traced per launch), and
    zinc_precompute_cache timed alone."""
    from paper_2408_07304_b200.dist import max_over_ranks, shard_range
    cfg = CONFIGS["C5"]
    ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale, device=dev.index or 0)
    sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
    out = {"workload": "C5", "ranks": world, "batches": {}}

    def timed(fn, n):
        fn()
        ts = []
        for _ in range(n):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    cache = {}
    for f, name in ((Z.COEFF, "coeff"), (Z.NTT, "ntt")):
        buf = ctx.empty_key()
        ms = timed(lambda: Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, f, out=buf), 5)
        cache[f] = buf
        out[f"cache_precompute_ms_{name}"] = ms
    free = torch.cuda.mem_get_info()[0]
    for B in batches:
        b0, b1 = shard_range(rank, world, B)
        nb = b1 - b0
        per = 2 * cfg.L * cfg.n * 8 + cfg.n // 2 * 8
        skip = float(nb * per > 0.85 * free)
        if max_over_ranks([skip], device=dev)[0] > 0:
            out["batches"][str(B)] = {"skipped": f"needs {nb * per / 2**30:.0f} GiB per rank"}
            continue
        zc = vn = 0.0
        if nb:
            z = torch.from_numpy(np.ascontiguousarray(slots_batch(cfg, b0, min(nb, 4096)))).to(dev)
            if nb > z.shape[0]:
                z = z.repeat((nb + z.shape[0] - 1) // z.shape[0], 1)[:nb].contiguous()
            ct = ctx.empty_ct(nb)
            fz = lambda: Z.zinc_encrypt_batch(ctx, cache[Z.COEFF], Z.COEFF, z, cfg.enc_seed, b0, out=ct)
            fv = lambda: Z.ckks_encrypt_batch(ctx, pk, Z.NTT, z, cfg.enc_seed, b0, out=ct)
            zc = timed(fz, reps)
            vn = timed(fv, reps)
            # device busy time: the library's per-kernel CUDA events, summed (no host gaps)
            busy = []
            for fn in (fz, fv):
                Z.profile_enable(True)
                fn()
                torch.cuda.synchronize()
                busy.append(sum(v[0] for v in Z.profile_read().values()))
                Z.profile_enable(False)
            zk, vk = busy
            del ct, z
            torch.cuda.empty_cache()
        else:
            zk = vk = 0.0
        zc, vn, zk, vk = max_over_ranks([zc, vn, zk, vk], device=dev)
        out["batches"][str(B)] = {"zinc_coeff_ms": zc, "zinc_coeff_ct_per_s": B / (zc / 1e3),
                                  "vanilla_ntt_ms": vn, "vanilla_ntt_ct_per_s": B / (vn / 1e3),
                                  "zinc_coeff_kernels_ms": zk, "vanilla_ntt_kernels_ms": vk,
                                  "ranks_active": min(world, B), "ranks_idle": max(0, world - B)}
    ctx.close()
    return out


def _timed(torch, fn, n):
    fn()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def other_configs(Z, torch, names=("C1", "C2", "C4"), reps=2):
    """The other BASELINE configs on one GPU (parity-tested in tests/): ct/s of the four
    encryption paths from slots and of batched decrypt+decode, device
    time with CUDA events (1 warm-up + `reps`, median).  Each config's full batch."""
    out = {}
    for name in names:
        cfg = CONFIGS[name]
        ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
        sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
        cache = {f: Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, f) for f in (Z.COEFF, Z.NTT)}
        B = cfg.batch
        z = slots_batch(cfg, 0, B)
        if cfg.complex_slots:
            z = np.stack([z.real, z.imag], axis=-1)
        zd = torch.from_numpy(np.ascontiguousarray(z)).cuda()
        ct = ctx.empty_ct(B)
        r = {"N": cfg.n, "L": cfg.L, "batch": B}
        for pname, fn in (
                ("zinc_coeff", lambda: Z.zinc_encrypt_batch(ctx, cache[Z.COEFF], Z.COEFF, zd, cfg.enc_seed, 0, out=ct)),
                ("zinc_ntt", lambda: Z.zinc_encrypt_batch(ctx, cache[Z.NTT], Z.NTT, zd, cfg.enc_seed, 0, out=ct)),
                ("vanilla_ntt", lambda: Z.ckks_encrypt_batch(ctx, pk, Z.NTT, zd, cfg.enc_seed, 0, out=ct)),
                ("vanilla_coeff", lambda: Z.ckks_encrypt_batch(ctx, pk, Z.COEFF, zd, cfg.enc_seed, 0, out=ct))):
            ms = _timed(torch, fn, reps)
            r[pname] = {"ms": ms, "ct_per_s": B / (ms / 1e3)}
        # f1: batched decrypt + decode of the last (vanilla COEFF) ciphertexts, checked
        ms = _timed(torch, lambda: Z.ckks_decrypt_batch(ctx, sk, Z.COEFF, ct), reps)
        _, st, zz = Z.ckks_decrypt_batch(ctx, sk, Z.COEFF, ct[:64])
        ref = slots_batch(cfg, 0, min(B, 64))
        err = float(np.max(np.abs(zz.cpu().numpy() - ref)))
        r["decrypt_decode_coeff"] = {"ms": ms, "ct_per_s": B / (ms / 1e3), "max_abs_err_64": err,
                                     "crt_ok": int(st.sum().item()) == 0, "tolerance": cfg.tolerance()}
        r["ok"] = r["decrypt_decode_coeff"]["crt_ok"] and err < cfg.tolerance()
        out[name] = r
        del ct, zd
        ctx.close()
        torch.cuda.empty_cache()
    return out


def paper_params(Z, torch, reps=2, cap=4096):
    """the paper's own parameters (N = 2^15, 881-bit Q, Delta = 2^55) on the
    Table 2 dataset shapes (synthetic stand-ins, workloads.py).  Zinc (COEFF) and vanilla (NTT
    form) from slots through the 128-bit plaintext path; up to `cap` messages per timed call,
    job time = count / rate.  The paper's single-threaded SEAL totals are context only."""
    paper_s = {"P_covid": (19.2, 8.2), "P_bitcoin": (62.2, 24.8), "P_hg38": (1983.6, 812.6)}  # Table 2
    out = {}
    for name in ("P_covid", "P_bitcoin", "P_hg38"):
        cfg = CONFIGS[name]
        ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
        sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
        cache = Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, Z.COEFF)
        B = min(cfg.batch, cap)
        zd = torch.from_numpy(np.ascontiguousarray(slots_batch(cfg, 0, B))).cuda()
        ct = ctx.empty_ct(B)
        zc = _timed(torch, lambda: Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, zd, cfg.enc_seed, 0, out=ct), reps)
        _, st, zz = Z.ckks_decrypt_batch(ctx, sk, Z.COEFF, ct[:8])
        err = float(np.max(np.abs(zz.cpu().numpy() - slots_batch(cfg, 0, 8))))
        vn = _timed(torch, lambda: Z.ckks_encrypt_batch(ctx, pk, Z.NTT, zd, cfg.enc_seed, 0, out=ct), reps)
        m128 = Z.ckks_encode_batch_wide(ctx, zd)  # the same plaintexts as 128-bit coefficients
        zi = _timed(torch, lambda: Z.zinc_encrypt_batch(ctx, cache, Z.COEFF, m128, cfg.enc_seed, 0, out=ct), reps)
        del m128
        rz, rv, ri = B / (zc / 1e3), B / (vn / 1e3), B / (zi / 1e3)
        peak = load_peaks()[0]
        ctb = 2 * cfg.L * cfg.n * 8
        out[name] = {"count": cfg.batch, "timed_batch": B, "zinc_coeff_ct_per_s": rz, "vanilla_ntt_ct_per_s": rv,
                     "zinc_coeff_hbm_frac": rz * (ctb + cfg.n // 2 * 8) / 1e9 / peak,
                     "zinc_coeff_i128_ct_per_s": ri, "zinc_coeff_i128_hbm_frac": ri * (ctb + cfg.n * 16) / 1e9 / peak,
                     "zinc_job_s": cfg.batch / rz, "vanilla_job_s": cfg.batch / rv,
                     "paper_seal_cpu_s": {"ckks": paper_s[name][0], "zinc": paper_s[name][1]},
                     "decrypt_ok": int(st.sum().item()) == 0 and err < 1e-4, "max_abs_err_8": err}
        del ct, zd
        ctx.close()
        torch.cuda.empty_cache()
    return out


def schemes(Z, torch, reps=2, B=4096, t=65537):
    """BFV (Eq. 12) and BGV (Eq. 13) at C3's ring and modulus, Zinc (COEFF and
    NTT form) and vanilla (NTT form) from int64 plaintexts mod t, with a decryption check."""
    cfg = CONFIGS["C3"]
    out = {"workload": "C3 ring, t = %d" % t, "batch": B}
    for name, scheme in (("BFV", 1), ("BGV", 2)):
        ctx = Z.Context(cfg.log_n, cfg.bits, 0, scheme=scheme, t=t)
        sk, _, pk = Z.zinc_keygen(ctx, cfg.key_seed)
        cache = {f: Z.zinc_precompute_cache(ctx, pk, cfg.cache_seed, f) for f in (Z.COEFF, Z.NTT)}
        gen = torch.Generator(device="cuda").manual_seed(5)
        m = torch.randint(0, t, (B, cfg.n), dtype=torch.int64, device="cuda", generator=gen)
        ct = ctx.empty_ct(B)
        r = {}
        for pname, fn in (
                ("zinc_coeff", lambda: Z.zinc_encrypt_batch(ctx, cache[Z.COEFF], Z.COEFF, m, cfg.enc_seed, 0, out=ct)),
                ("zinc_ntt", lambda: Z.zinc_encrypt_batch(ctx, cache[Z.NTT], Z.NTT, m, cfg.enc_seed, 0, out=ct)),
                ("vanilla_ntt", lambda: Z.ckks_encrypt_batch(ctx, pk, Z.NTT, m, cfg.enc_seed, 0, out=ct))):
            ms = _timed(torch, fn, reps)
            r[pname] = {"ms": ms, "ct_per_s": B / (ms / 1e3)}
        coeff, st, _ = Z.ckks_decrypt_batch(ctx, sk, Z.NTT, ct[:64])
        r["decrypt_ok"] = bool(torch.equal(coeff, m[:64])) and int(st.sum().item()) == 0
        out[name] = r
        del ct, m
        ctx.close()
        torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="messages split over all ranks as [r B/P, (r+1) B/P) (default: the config's batch; "
                         "strong scaling, SURVEY.md 8(e))")
    ap.add_argument("--batch", type=int, default=0, help="messages per GPU instead (weak scaling)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: CUDA tensors through the host; tests)")
    ap.add_argument("--paths", default=",".join(PATHS))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-oracle-suite", action="store_true", help="skip the per-config oracle runs (8(d))")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 batch sweep")
    ap.add_argument("--c5-batches", default="1,16,256,4096,65536", help="C5 sweep batch sizes")
    ap.add_argument("--no-others", action="store_true", help="skip the C1/C2/C4 single-GPU lines")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_2408_07304_b200 as Z
    from paper_2408_07304_b200.dist import broadcast_words, max_over_ranks, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    gpu = local % torch.cuda.device_count()  # one rank per GPU; gloo tests may share one
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    def sum_over_ranks(x):
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t)
        return float(t.item())

    paths = [p for p in args.paths.split(",") if p]
    if args.batch:
        B_global, scaling = args.batch * world, "weak"
    else:
        B_global, scaling = args.global_batch or cfg.batch, "strong"
    b0, b1 = shard_range(rank, world, B_global)
    B = b1 - b0  # this rank's messages [b0, b1), msg_base = b0: bit-identical for any P
    ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale, device=gpu)
    stream = torch.cuda.current_stream()

    # keys + cache on rank 0, broadcast once; every rank also regenerates
    # them locally and checks the broadcast copies bit for bit.
    sk, _, pk_local = Z.zinc_keygen(ctx, cfg.key_seed)
    cache_local = {f: Z.zinc_precompute_cache(ctx, pk_local, cfg.cache_seed, f) for f in (Z.COEFF, Z.NTT)}
    pk = pk_local.clone()
    cache = {f: c.clone() for f, c in cache_local.items()}
    bcast_ok, bcast_ms = True, 0.0
    if world > 1:
        if rank != 0:  # receivers start from garbage so the check is meaningful
            for t in (pk, cache[Z.COEFF], cache[Z.NTT]):
                t.fill_(7)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        broadcast_words([pk, cache[Z.COEFF], cache[Z.NTT]], src=0)
        torch.cuda.synchronize()
        bcast_ms = 1e3 * (time.perf_counter() - t0)
        ok = all(torch.equal(a, b) for a, b in ((pk, pk_local), (cache[0], cache_local[0]), (cache[1], cache_local[1])))
        bcast_ok = sum_over_ranks(0 if ok else 1) == 0

    # inputs: this rank's messages, resident in HBM
    t0 = time.time()
    slots_h = slots_batch(cfg, b0, B)
    if cfg.complex_slots:
        slots_h = np.stack([slots_h.real, slots_h.imag], axis=-1)
    slots = torch.from_numpy(np.ascontiguousarray(slots_h)).to(dev)
    ct = ctx.empty_ct(B)
    log(f"[rank {rank}] inputs ready ({time.time() - t0:.1f}s): messages [{b0}, {b1}), "
        f"ct buffer {ct.numel() * 8 / 2**30:.1f} GiB")

    def run(path):
        if B == 0:
            return
        if path == "zinc_coeff":
            Z.zinc_encrypt_batch(ctx, cache[Z.COEFF], Z.COEFF, slots, cfg.enc_seed, b0, out=ct)
        elif path == "zinc_ntt":
            Z.zinc_encrypt_batch(ctx, cache[Z.NTT], Z.NTT, slots, cfg.enc_seed, b0, out=ct)
        elif path == "vanilla_ntt":
            Z.ckks_encrypt_batch(ctx, pk, Z.NTT, slots, cfg.enc_seed, b0, out=ct)
        elif path == "vanilla_coeff":
            Z.ckks_encrypt_batch(ctx, pk, Z.COEFF, slots, cfg.enc_seed, b0, out=ct)

    # validity gate: every path's output, from the exact call the timed region
    # makes, decrypts within tolerance with a consistent CRT, sampled at the first and last
    # message of every 256-message block of every rank's shard -- so every chunk of every
    # chunk chain (Zinc COEFF: 256-message chunks; transform paths: 16-wave chunks) and both
    # halves of C3's A13 mix
    validity = {}
    probe_idx = sorted(set([b for k in range(0, B, 256) for b in (k, min(B, k + 256) - 1)]))
    pidx = torch.tensor(probe_idx, dtype=torch.long, device=dev)
    ref_all = (slots_h[probe_idx, :, 0] + 1j * slots_h[probe_idx, :, 1]) if cfg.complex_slots else slots_h[probe_idx]
    failed = 0
    for p in paths:
        run(p)
        ok, crt, err = True, True, 0.0
        if probe_idx:
            form = Z.COEFF if p.endswith("coeff") else Z.NTT
            _, st, z = Z.ckks_decrypt_batch(ctx, sk, form, ct.index_select(0, pidx).contiguous())
            err = float(np.max(np.abs(z.cpu().numpy() - ref_all)))
            crt = int(st.sum().item()) == 0
            ok = crt and err < cfg.tolerance()
        err = max_over_ranks([err], device=dev)[0]
        bad = sum_over_ranks(0 if ok else 1)
        validity[p] = {"crt_ok": bad == 0 and crt, "max_abs_err": err, "ok": bad == 0, "tolerance": cfg.tolerance(),
                       "sampled": int(sum_over_ranks(len(probe_idx)))}
        failed += bad > 0
        if bad:
            log(f"validity gate failed for {p}: {validity[p]}")
    if failed:
        sys.exit(3)
    validity["sampled_indices_rank0"] = [b0 + b for b in probe_idx] if rank == 0 else None

    for _ in range(args.warmup):
        for p in paths:
            run(p)
    torch.cuda.synchronize()

    # int-peak microkernel (K11) per butterfly variant: the denominators of the transform paths
    sink = torch.zeros(2, dtype=torch.uint64, device=dev)
    nr_ok = max(ctx.q) < (1 << 58)
    k11 = {}
    for v in ((1, 2, 3) if nr_ok else (2, 3)):
        Z.zinc_int_peak(ctx, 148 * 8, 200, sink, variant=v)
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            bf = Z.zinc_int_peak(ctx, 148 * 8, 4000, sink, variant=v)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, bf / (e0.elapsed_time(e1) / 1e3))
        k11[v] = best
    fwd_v = 1 if nr_ok else 2  # the forward butterfly the CKKS transform kernels run at this modulus

    # ---------------- timed region
    ev = {p: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)] for p in paths}
    clocks = ClockSampler(gpu)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.25)
    Z.launch_count_reset()
    for k in range(args.steps):
        for p in paths:
            ev[p][k][0].record(stream)
            run(p)
            ev[p][k][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = Z.launch_count()
    clk = clocks.stop()
    # Per-kernel device times come from one extra, untimed step with the library's launch
    # tracing on: its events sit between launches on the stream, which would break the
    # programmatic dependent launches of the slot pipeline inside the timed region.
    prof, prof_path = {}, {}
    for p in paths:
        Z.profile_enable(True)
        run(p)
        torch.cuda.synchronize()
        prof_path[p] = Z.profile_read()
        Z.profile_enable(False)
        for k, v in prof_path[p].items():
            a0, a1 = prof.get(k, (0.0, 0))
            prof[k] = (a0 + v[0] * args.steps, a1 + v[1] * args.steps)

    seg_local = {p: sum(a.elapsed_time(b) for a, b in ev[p]) / args.steps for p in paths}  # ms per step
    seg = dict(zip(paths, max_over_ranks([seg_local[p] for p in paths], device=dev)))
    launches = int(sum_over_ranks(launches))
    path_out = {p: {"ct_per_s": B_global / (seg[p] / 1e3), "ms": seg[p]} for p in paths}

    peak, peak_src = load_peaks()
    result = None
    if rank == 0:
        bpc = bytes_per_ct(cfg, "slots")
        kbytes = bytes_per_ct(cfg, "int64")
        zk_ms, zk_n = prof.get("zinc_coeff_kernel", (0.0, 0))  # the dominant kernel of the value path
        roof = None
        if zk_n:
            per_launch_ms = zk_ms / zk_n
            msgs_per_launch = B * args.steps / zk_n
            achieved = msgs_per_launch * kbytes / (per_launch_ms / 1e3) / 1e9
            roof = {"bound": "hbm", "kernel": "zinc_coeff_kernel", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                    "algorithmic_bytes_per_ct": kbytes, "msgs_per_launch": msgs_per_launch,
                    "launch_ms": per_launch_ms,
                    "kernel_share_of_zinc_segment": zk_ms / args.steps / seg_local["zinc_coeff"]
                    if "zinc_coeff" in seg_local else None,
                    "kernel_timing": "CUDA events around each launch of one extra traced step (on the launch "
                                     "stream), scaled to the timed steps; rank 0's own launches"}
            tr = os.path.join(ROOT, "profiles", "ncu_traffic.json")
            if os.path.exists(tr):
                t = json.load(open(tr)).get("zinc_coeff_kernel")
                if t and t.get("config") == cfg.name:
                    roof["traffic"] = t["dram_bytes_per_msg"] * msgs_per_launch
                    roof["traffic_source"] = "profiles/ncu_traffic.json (ncu --set full, per message, scaled)"
        alu = {}
        sm_mhz = clk["sm_mhz"] or 1965.0
        for p, kname in (("zinc_ntt", "zinc_ntt_kernel"), ("vanilla_ntt", "vanilla_kernel"),
                         ("vanilla_coeff", "vanilla_kernel")):
            if p not in seg_local or B == 0:
                continue
            nf, ni = path_transforms(cfg, p)
            # the path's own peak: its forward and inverse butterflies at their K11 rates
            peak_p = (nf + ni) / (nf / k11[fwd_v] + ni / k11[3])
            pd = (nf + ni) / (nf / alu_peak_derived(sm_mhz, BFLY[fwd_v][2]) + ni / alu_peak_derived(sm_mhz, BFLY[3][2]))
            kms = prof_path[p].get(kname, (0.0, 0))[0]
            bfc = butterflies_per_ct(cfg, p)
            ach = bfc * B / (seg_local[p] / 1e3)
            kach = bfc * B / (kms / 1e3) if kms else ach
            alu[p] = {"bound": "alu", "kernel": kname, "achieved": kach / 1e9, "peak": peak_p / 1e9,
                      "unit": "Gbutterfly/s", "frac": kach / peak_p, "achieved_path": ach / 1e9,
                      "frac_path": ach / peak_p, "peak_derived": pd / 1e9, "frac_of_derived": kach / pd,
                      "butterflies_per_ct": bfc, "transforms_per_ct": {"forward": nf, "inverse": ni},
                      "peak_source": f"measured K11 int_peak_kernel with the path's own butterflies: {nf} x "
                                     f"{BFLY[fwd_v][0]} + {ni} x {BFLY[3][0]} per ct (harmonic mix); peak_derived: "
                                     f"148 SMs x sm_mhz x 64 fma-pipe lanes/clk / SASS fma ops per butterfly "
                                     f"({BFLY[fwd_v][2]} {BFLY[fwd_v][0]}, {BFLY[3][2]} {BFLY[3][0]})"}
        multi = "" if world == 1 else f", {world} ranks"
        result = {
            "metric": METRIC,
            "value": path_out["zinc_coeff"]["ct_per_s"] if "zinc_coeff" in path_out else None,
            "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sum(seg.values()),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (workloads.py seeded slots; paper datasets not in container)",
            "config": {"workload": cfg.name, "N": cfg.n, "L": cfg.L, "bits": list(cfg.bits),
                       "log_scale": cfg.log_scale, "global_batch": B_global, "batch_rank0": B,
                       "shard": "rank r: messages [r B/P, (r+1) B/P), msg_base = r B/P",
                       "input": "f64 slots in HBM", "value_path": "zinc_coeff (encode + Zinc add/inject, COEFF form)",
                       "l2": "inputs and outputs (GiB) exceed the 126 MB L2; no flush",
                       "parallelism": f"dp{world} (message-sharded, {args.backend if world > 1 else 'no'} broadcast "
                                      f"of pk + caches{multi})"},
            "paths": path_out,
            "zinc_vs_vanilla": {
                "coeff_form": path_out["zinc_coeff"]["ct_per_s"] / path_out["vanilla_coeff"]["ct_per_s"]
                if {"zinc_coeff", "vanilla_coeff"} <= set(path_out) else None,
                "ntt_form": path_out["zinc_ntt"]["ct_per_s"] / path_out["vanilla_ntt"]["ct_per_s"]
                if {"zinc_ntt", "vanilla_ntt"} <= set(path_out) else None},
            "hbm_frac_step": (bpc * B / (seg_local["zinc_coeff"] / 1e3) / 1e9) / peak
            if "zinc_coeff" in seg_local and B else None,
            "roofline": roof,
            "roofline_alu": alu,
            "k11_gbfly": {BFLY[v][0]: r / 1e9 for v, r in k11.items()},
            "kernels": {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps}
                        for k, v in prof.items()},
            "gpu_launches": launches,
            "clocks": clk,
            "validity": validity,
            "broadcast_ok": bcast_ok,
            "broadcast_ms": bcast_ms if world > 1 else None,
        }
        if world > 1:
            result["multi_gpu"] = {"backend": args.backend, "ranks": world, "hardware": "measured" if
                                   args.backend == "nccl" else "logic test (gloo; ranks may share a GPU)"}

    if "vanilla_coeff" in paths:
        # batched decrypt + decode (Eq. 10, CRT check on every limb) of the
        # step's last output (vanilla COEFF form), device-timed like the paths, every rank
        dms = _timed(torch, lambda: Z.ckks_decrypt_batch(ctx, sk, Z.COEFF, ct), 3) if B else 0.0
        dk = 0.0
        if B:
            Z.profile_enable(True)
            Z.ckks_decrypt_batch(ctx, sk, Z.COEFF, ct)
            torch.cuda.synchronize()
            dk = Z.profile_read().get("decrypt_kernel", (0.0, 0))[0]
            Z.profile_enable(False)
        dmax = max_over_ranks([dms], device=dev)[0]
        if rank == 0:
            dpeak = 2 / (1 / k11[2] + 1 / k11[3])
            dbf = butterflies_per_ct(cfg, "decrypt_coeff")
            result["decrypt_decode"] = {"form": "COEFF", "ms": dmax, "ct_per_s": B_global / (dmax / 1e3),
                                        "transforms_per_ct": 2 * cfg.L,
                                        "note": "x = c1 + c2 s on every limb (NTT + INTT per limb), CRT check, "
                                                "FP64 decode"}
            result["roofline_alu"]["decrypt_coeff"] = {
                "bound": "alu", "kernel": "decrypt_kernel", "achieved": dbf * B / (dk / 1e3) / 1e9 if dk else None,
                "peak": dpeak / 1e9, "unit": "Gbutterfly/s", "frac": dbf * B / (dk / 1e3) / dpeak if dk else None,
                "butterflies_per_ct": dbf, "transforms_per_ct": {"forward": cfg.L, "inverse": cfg.L},
                "peak_source": "measured K11 with the kernel's butterflies: L x ct_bfly_a + L x gs_bfly per ct"}
    # aggregation of each rank's shard (Eq. 2, HBM-bound read of every ciphertext)
    agg = ctx.empty_key()
    ams = _timed(torch, lambda: Z.zinc_ct_sum_batch(ctx, ct, out=agg), 3) if B else 0.0
    amax = max_over_ranks([ams], device=dev)[0]
    if rank == 0:
        rb = B * 2 * cfg.L * cfg.n * 8
        result["aggregate"] = {"ms": amax, "ct_per_s": B_global / (amax / 1e3), "GBps_rank0": rb / (ams / 1e3) / 1e9,
                               "frac_hbm_rank0": rb / (ams / 1e3) / 1e9 / peak, "batch_rank0": B,
                               "note": "zinc_ct_sum_batch over each rank's last output (read 2 L N 8 B per ct)"}
    if not args.no_c5:
        del ct
        ct = None
        torch.cuda.empty_cache()
        c5 = c5_sweep(Z, torch, dev, rank, world, batches=tuple(int(x) for x in args.c5_batches.split(",") if x))
        if rank == 0:
            result["c5"] = c5
    if rank == 0 and world == 1 and not args.no_others:
        if ct is not None:
            del ct
            ct = None
            torch.cuda.empty_cache()
        result["other_configs"] = other_configs(Z, torch)
        result["paper_params"] = paper_params(Z, torch)
        result["schemes"] = schemes(Z, torch)

    # ---------------- end to end through the host-buffer API, every rank on its shard
    if not args.no_e2e:
        import psutil
        per_msg = (slots_h[0].nbytes if B else 0) + 2 * cfg.L * cfg.n * 8
        budget = 0.6 * psutil.virtual_memory().available / max(1, world)
        Be = int(min(B, budget // per_msg))
        if Be:
            pt_h = torch.from_numpy(np.ascontiguousarray(slots_h[:Be])).pin_memory()
            ct_h = torch.empty((Be, 2, cfg.L, cfg.n), dtype=torch.uint64, pin_memory=True)
            Z.zinc_encrypt_batch_host(ctx, 0, cache[Z.COEFF], Z.COEFF, pt_h, cfg.enc_seed, b0, ct_h)
        ts = []
        for _ in range(args.e2e_steps):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            if Be:
                Z.zinc_encrypt_batch_host(ctx, 0, cache[Z.COEFF], Z.COEFF, pt_h, cfg.enc_seed, b0, ct_h)
            ts.append(time.perf_counter() - t0)
        tt = max_over_ranks([min(ts)], device=dev)[0]
        be_tot = sum_over_ranks(Be)
        if rank == 0:
            result["e2e"] = {"value": be_tot / tt, "unit": UNIT,
                             "h2d_bytes_per_step": int(pt_h.numel() * 8 if Be else 0),
                             "d2h_bytes_per_step": int(ct_h.numel() * 8 if Be else 0),
                             "bytes_scope": "rank 0's per-step copies", "global_batch": int(be_tot),
                             "api": "zinc_encrypt_batch_host (pinned host in/out, 2 streams)",
                             "path": "zinc_coeff", "timer": "host perf_counter around the blocking call on every "
                             f"rank after a barrier, max over ranks, best of {args.e2e_steps}"}
        if Be:
            del pt_h, ct_h

    # ---------------- the oracle beside it (rank 0's host cores; the other ranks wait)
    if rank == 0 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        r, n, w, vr, vn = oracle_rate(cfg, args.cpu_seconds, threads)
        result["cpu_baseline"] = {"value": r, "unit": UNIT, "cores": threads, "kind": "oracle",
                                  "sample": f"{n} {cfg.name} Zinc COEFF encryptions from slots (oracle encode + "
                                            f"Enc_z) in {w:.1f} s; vanilla NTT-form {vn} msgs: {vr:.2f} ct/s",
                                  "vanilla_ct_per_s": vr, "cpu": cpu_model()}
        if not args.no_oracle_suite:
            result["cpu_baseline"]["suite"] = oracle_suite(sorted({1, threads}))
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
