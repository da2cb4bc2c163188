"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Bar (BASELINE.json north_star): ciphertext words bit-exact given the same seed
and the same int64 plaintext; encode within +-1 per coefficient (floating point,
C-6 / reading A9); decoded slots within 1e-4 at 2^40, 1e-3 at 2^30.
"""
import numpy as np
import pytest
import torch

from workloads import CONFIGS, int_plaintexts, message_slots, slots_batch

pytestmark = pytest.mark.gpu

NTT, COEFF = 0, 1


def np64(t):
    return t.cpu().numpy()


def dev_u64(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64)).cuda()


def dev_i64(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).cuda()


@pytest.fixture(scope="module")
def Z():
    import paper_2408_07304_b200 as Z
    assert torch.cuda.is_available()
    return Z


class Setup:
    def __init__(self, Z, orc, cfg):
        self.cfg = cfg
        self.ctx = Z.Context(cfg.log_n, cfg.bits, cfg.log_scale)
        self.P = orc.Params.make(cfg.log_n, cfg.bits, cfg.log_scale)
        self.sk, self.skc, self.pk = Z.zinc_keygen(self.ctx, cfg.key_seed)
        self.o_sk, self.o_sk_ntt, self.o_pk = orc.keygen(self.P, cfg.key_seed)
        self.cache = {f: Z.zinc_precompute_cache(self.ctx, self.pk, cfg.cache_seed, f) for f in (NTT, COEFF)}
        torch.cuda.synchronize()


_setups = {}


def setup_for(Z, orc, name):
    if name not in _setups:
        _setups[name] = Setup(Z, orc, CONFIGS[name])
    return _setups[name]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_params_match_oracle(Z, orc, name):
    s = setup_for(Z, orc, name)
    assert s.ctx.q == [int(x) for x in s.P.q]
    assert s.ctx.psi == [int(x) for x in s.P.psi]


@pytest.mark.parametrize("tag", [1, 2, 3, 4, 5, 6, 7, 8])
def test_sampler_streams_bit_exact(Z, orc, tag):
    s = setup_for(Z, orc, "C3")
    n = 4100  # ragged: not a multiple of the 4-per-block ternary layout
    for seed, msg, limb in [(1, 0, 0), (0xDEADBEEFCAFEF00D, (1 << 32) + 5, 3), (7, (1 << 64) - 1, 7)]:
        got = np64(Z.zinc_debug_sample(s.ctx, tag, seed, msg, limb, n))
        if tag == 3:
            want = orc.sample_uniform(seed, msg, tag, limb, int(s.P.q[limb]), n)
        elif tag in (1, 4):
            want = orc.sample_ternary(seed, msg, tag, n)
        else:
            want = orc.sample_cbd(seed, msg, tag, n)
        assert np.array_equal(got, want), (tag, seed, msg, limb)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_ntt_bit_exact(Z, orc, name):
    s = setup_for(Z, orc, name)
    rng = np.random.default_rng(11)
    count = 3
    x = np.stack([np.stack([rng.integers(0, int(q), s.P.n, dtype=np.uint64) for q in s.P.q]) for _ in range(count)])
    d = dev_u64(x)
    Z.zinc_ntt_forward(s.ctx, d)
    fwd = np64(d)
    for c in range(count):
        assert np.array_equal(fwd[c], orc.ntt_limbs(s.P, x[c]))
    Z.zinc_ntt_inverse(s.ctx, d)
    assert np.array_equal(np64(d), x)
    # edge values: all q-1, all 0
    e = np.stack([np.full(s.P.n, int(q) - 1, dtype=np.uint64) for q in s.P.q])[None]
    d = dev_u64(e)
    Z.zinc_ntt_forward(s.ctx, d)
    assert np.array_equal(np64(d)[0], orc.ntt_limbs(s.P, e[0]))


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_keygen_and_cache_bit_exact(Z, orc, name):
    s = setup_for(Z, orc, name)
    assert np.array_equal(np64(s.skc).astype(np.int64), s.o_sk)
    assert np.array_equal(np64(s.sk), s.o_sk_ntt)
    assert np.array_equal(np64(s.pk), s.o_pk)
    for f in (NTT, COEFF):
        assert np.array_equal(np64(s.cache[f]), orc.precompute_cache(s.P, s.o_pk, s.cfg.cache_seed, f))


def _check_msgs(orc, s, path, form, m, got, seed, msg_base, idx):
    key = s.o_pk if path == "vanilla" else orc.precompute_cache(s.P, s.o_pk, s.cfg.cache_seed, form)
    for b in idx:
        if path == "vanilla":
            want = orc.vanilla_encrypt(s.P, key, m[b], seed, msg_base + b, form)
        else:
            want = orc.zinc_encrypt(s.P, key, form, m[b], seed, msg_base + b)
        assert np.array_equal(got[b], want), (path, form, b)


@pytest.mark.parametrize("path", ["zinc", "vanilla"])
@pytest.mark.parametrize("form", [NTT, COEFF])
def test_encrypt_int64_c1_all_messages(Z, orc, path, form):
    """C1 in full: all 256 messages bit-exact."""
    s = setup_for(Z, orc, "C1")
    B = s.cfg.batch
    m = int_plaintexts(s.cfg.log_n, B, seed=1, bound_bits=34)
    seed, base = s.cfg.enc_seed, 1000
    if path == "zinc":
        ct = Z.zinc_encrypt_batch(s.ctx, s.cache[form], form, dev_i64(m), seed, base)
    else:
        ct = Z.ckks_encrypt_batch(s.ctx, s.pk, form, dev_i64(m), seed, base)
    _check_msgs(orc, s, path, form, m, np64(ct), seed, base, range(B))


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
@pytest.mark.parametrize("path", ["zinc", "vanilla"])
@pytest.mark.parametrize("form", [NTT, COEFF])
def test_encrypt_int64_sampled(Z, orc, name, path, form):
    """Ragged batch (37 messages, not a multiple of any tile), sampled messages."""
    s = setup_for(Z, orc, name)
    B = 37
    m = int_plaintexts(s.cfg.log_n, B, seed=2, bound_bits=50)
    m[3, :5] = [np.iinfo(np.int64).max, np.iinfo(np.int64).min + 1, -(1 << 62), (1 << 61) + 12345, -1]  # slow reduce path
    seed, base = 0x123456789, (1 << 32) - 20  # message indices cross the 2^32 counter word
    if path == "zinc":
        ct = Z.zinc_encrypt_batch(s.ctx, s.cache[form], form, dev_i64(m), seed, base)
    else:
        ct = Z.ckks_encrypt_batch(s.ctx, s.pk, form, dev_i64(m), seed, base)
    _check_msgs(orc, s, path, form, m, np64(ct), seed, base, [0, 3, 19, 20, 36])


@pytest.mark.parametrize("split", [0, 2])
@pytest.mark.parametrize("name", ["C3", "C4"])
def test_both_transform_kernel_families_bit_exact(Z, orc, name, split):
    """Both kernel families at N >= 2^14 (2-CTA parity split, S-CTA clusters; the default
    picks one per path): every transform path and decryption bit-exact on a ragged batch."""
    s = setup_for(Z, orc, name)
    B = 21
    m = int_plaintexts(s.cfg.log_n, B, seed=12, bound_bits=48)
    seed, base = 0x5151, 777
    old = Z.tune(Z.TUNE_SPLIT, split)
    try:
        cts = {("zinc", NTT): Z.zinc_encrypt_batch(s.ctx, s.cache[NTT], NTT, dev_i64(m), seed, base),
               ("vanilla", NTT): Z.ckks_encrypt_batch(s.ctx, s.pk, NTT, dev_i64(m), seed, base),
               ("vanilla", COEFF): Z.ckks_encrypt_batch(s.ctx, s.pk, COEFF, dev_i64(m), seed, base)}
        dec = {f: Z.ckks_decrypt_batch(s.ctx, s.sk, f, cts[("vanilla", f)], slots=False) for f in (NTT, COEFF)}
        torch.cuda.synchronize()
    finally:
        Z.tune(Z.TUNE_SPLIT, old)
    for (path, form), ct in cts.items():
        _check_msgs(orc, s, path, form, m, np64(ct), seed, base, [0, 10, 20])
    for f, (coeff, st, _) in dec.items():
        assert (np64(st) == 0).all()
        c = np64(coeff)
        for b in (0, 20):
            x, ost = orc.decrypt(s.P, s.o_sk_ntt, np64(cts[("vanilla", f)][b]), f)
            assert ost == 0 and np.array_equal(c[b], x)


@pytest.mark.parametrize("name", ["C3", "C4", "C2"])
@pytest.mark.parametrize("B", [1, 2, 5])
def test_small_batch_latency_paths_bit_exact(Z, orc, name, B):
    """Latency paths for a handful of messages (C5 batches 1 and 16): the 1024-thread encode,
    the finer Zinc COEFF tiles, and the transform-split Zinc NTT / vanilla NTT launches with
    the combine kernel -- bit-exact against the oracle on the GPU-encoded plaintexts."""
    s = setup_for(Z, orc, name)
    cfg = s.cfg
    z = slots_batch(cfg, 3, B)
    zz = np.stack([z.real, z.imag], axis=-1) if cfg.complex_slots else z
    zd = torch.from_numpy(np.ascontiguousarray(zz)).cuda()
    m = np64(Z.ckks_encode_batch(s.ctx, zd))
    seed, base = 99, 4242
    for path, form in (("zinc", COEFF), ("zinc", NTT), ("vanilla", NTT), ("vanilla", COEFF)):
        if path == "zinc":
            ct = Z.zinc_encrypt_batch(s.ctx, s.cache[form], form, zd, seed, base)
        else:
            ct = Z.ckks_encrypt_batch(s.ctx, s.pk, form, zd, seed, base)
        _check_msgs(orc, s, path, form, m, np64(ct), seed, base, sorted({0, B - 1}))
        _, st, zdec = Z.ckks_decrypt_batch(s.ctx, s.sk, form, ct)
        assert (np64(st) == 0).all()
        assert np.max(np.abs(zdec.cpu().numpy() - z)) < cfg.tolerance()


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_split_rendezvous_repeatability(Z, orc, name):
    """The S-CTA kernels' DSMEM exchanges under load: thousands of cluster rendezvous per call.
    COEFF-form decryption (forward exchange that reads every input before overwriting its own
    share) and the encryptions are repeated and must be identical and CRT-consistent every time
    (a missing load-completion before the buffer-free rendezvous failed ~1 in 7000 here)."""
    s = setup_for(Z, orc, name)
    B = 2048 if name == "C3" else 512
    z = torch.from_numpy(np.ascontiguousarray(slots_batch(s.cfg, 0, B) if not s.cfg.complex_slots else np.stack(
        [slots_batch(s.cfg, 0, B).real, slots_batch(s.cfg, 0, B).imag], axis=-1))).cuda()
    ct = Z.ckks_encrypt_batch(s.ctx, s.pk, COEFF, z, 8, 0)
    for _ in range(4):
        assert torch.equal(Z.ckks_encrypt_batch(s.ctx, s.pk, COEFF, z, 8, 0), ct)
        _, st, _ = Z.ckks_decrypt_batch(s.ctx, s.sk, COEFF, ct, slots=False)
        assert int(st.sum()) == 0


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_encode_within_one(Z, orc, name):
    s = setup_for(Z, orc, name)
    cfg = s.cfg
    B = 6
    z = slots_batch(cfg, 0, B) if name != "C3" else np.stack(
        [message_slots(cfg, b) for b in (0, 1, cfg.batch - 2, cfg.batch - 1, 5, 9000)])
    m = np64(Z.ckks_encode_batch(s.ctx, torch.from_numpy(np.ascontiguousarray(z)).cuda()))
    for b in range(B):
        want = orc.encode(z[b], cfg.log_n, cfg.log_scale)
        assert np.max(np.abs(m[b] - want)) <= 1
    if name == "C1":
        want = orc.encode_definition(z[0], cfg.log_n, cfg.log_scale)
        assert np.max(np.abs(m[0] - want)) <= 1


def test_encode_complex_slots(Z, orc):
    s = setup_for(Z, orc, "C2")
    rng = np.random.default_rng(5)
    z = rng.uniform(-1, 1, (3, s.P.n // 2)) + 1j * rng.uniform(-1, 1, (3, s.P.n // 2))
    zz = np.stack([z.real, z.imag], axis=-1)
    m = np64(Z.ckks_encode_batch(s.ctx, torch.from_numpy(np.ascontiguousarray(zz)).cuda()))
    for b in range(3):
        assert np.max(np.abs(m[b] - orc.encode(z[b], s.P.log_n, s.P.log_scale))) <= 1


@pytest.mark.parametrize("name", ["C1", "C3", "C4"])
@pytest.mark.parametrize("path", ["zinc", "vanilla"])
@pytest.mark.parametrize("form", [NTT, COEFF])
def test_slots_to_ciphertext_and_decrypt(Z, orc, name, path, form):
    """Slots in: the ciphertext equals the oracle's encryption of the GPU's encoded m
    bit for bit; decrypt status 0, coeff = oracle decrypt, slots within tolerance."""
    s = setup_for(Z, orc, name)
    cfg = s.cfg
    B = 12
    z = slots_batch(cfg, 0, B)
    zd = torch.from_numpy(z).cuda()
    m_gpu = np64(Z.ckks_encode_batch(s.ctx, zd))
    seed = cfg.enc_seed
    if path == "zinc":
        ct = Z.zinc_encrypt_batch(s.ctx, s.cache[form], form, zd, seed, 0)
    else:
        ct = Z.ckks_encrypt_batch(s.ctx, s.pk, form, zd, seed, 0)
    got = np64(ct)
    _check_msgs(orc, s, path, form, m_gpu, got, seed, 0, [0, 7, 11])
    coeff, status, slots = Z.ckks_decrypt_batch(s.ctx, s.sk, form, ct)
    assert (np64(status) == 0).all()
    coeff = np64(coeff)
    for b in (0, 7, 11):
        x, st = orc.decrypt(s.P, s.o_sk_ntt, got[b], form)
        assert st == 0 and np.array_equal(coeff[b], x)
    err = np.max(np.abs(slots.cpu().numpy() - z))
    assert err < cfg.tolerance(), err


@pytest.mark.parametrize("name", ["C1", "C4"])
def test_decrypt_wrong_key_flags_crt(Z, orc, name):
    s = setup_for(Z, orc, name)
    z = torch.from_numpy(slots_batch(s.cfg, 0, 4)).cuda()
    ct = Z.zinc_encrypt_batch(s.ctx, s.cache[COEFF], COEFF, z, 1, 0)
    other, _, _ = Z.zinc_keygen(s.ctx, 999)
    _, status, _ = Z.ckks_decrypt_batch(s.ctx, other, COEFF, ct, slots=False)
    assert (np64(status) == 1).all()


@pytest.mark.parametrize("name", ["C1", "C4"])
def test_decode_matches_oracle(Z, orc, name):
    s = setup_for(Z, orc, name)
    z = torch.from_numpy(slots_batch(s.cfg, 3, 2)).cuda()
    ct = Z.ckks_encrypt_batch(s.ctx, s.pk, NTT, z, 4, 0)
    coeff, status, slots = Z.ckks_decrypt_batch(s.ctx, s.sk, NTT, ct)
    c = np64(coeff)
    for b in range(2):
        want = orc.decode(c[b], s.P.log_n, s.P.log_scale)
        assert np.max(np.abs(slots[b].cpu().numpy() - want)) < 1e-9


def test_forms_related_by_one_ntt(Z, orc):
    s = setup_for(Z, orc, "C2")
    m = dev_i64(int_plaintexts(s.cfg.log_n, 5, seed=3))
    for path in ("zinc", "vanilla"):
        if path == "zinc":
            a = Z.zinc_encrypt_batch(s.ctx, s.cache[COEFF], COEFF, m, 9, 0)
            b = Z.zinc_encrypt_batch(s.ctx, s.cache[NTT], NTT, m, 9, 0)
        else:
            a = Z.ckks_encrypt_batch(s.ctx, s.pk, COEFF, m, 9, 0)
            b = Z.ckks_encrypt_batch(s.ctx, s.pk, NTT, m, 9, 0)
        Z.zinc_ntt_forward(s.ctx, a.view(-1, s.ctx.L, s.ctx.n))
        assert torch.equal(a, b)


def test_sharding_is_bit_identical(Z, orc):
    """msg_base = global offset: two half-batches equal one batch (any P)."""
    s = setup_for(Z, orc, "C2")
    m = dev_i64(int_plaintexts(s.cfg.log_n, 40, seed=4))
    for fn, key in ((Z.zinc_encrypt_batch, s.cache[COEFF]),):
        full = fn(s.ctx, key, COEFF, m, 77, 500)
        a = fn(s.ctx, key, COEFF, m[:13].contiguous(), 77, 500)
        b = fn(s.ctx, key, COEFF, m[13:].contiguous(), 77, 513)
        assert torch.equal(full, torch.cat([a, b]))
    full = Z.ckks_encrypt_batch(s.ctx, s.pk, NTT, m, 77, 500)
    a = Z.ckks_encrypt_batch(s.ctx, s.pk, NTT, m[:13].contiguous(), 77, 500)
    b = Z.ckks_encrypt_batch(s.ctx, s.pk, NTT, m[13:].contiguous(), 77, 513)
    assert torch.equal(full, torch.cat([a, b]))


def test_batch_zero_and_bad_arguments(Z, orc):
    s = setup_for(Z, orc, "C1")
    m0 = torch.zeros((0, s.ctx.n), dtype=torch.int64, device="cuda")
    Z.zinc_encrypt_batch(s.ctx, s.cache[COEFF], COEFF, m0, 1, 0, out=s.ctx.empty_ct(0))  # no-op
    m1 = torch.zeros((1, s.ctx.n), dtype=torch.int64, device="cuda")
    with pytest.raises(Z.ZincError):
        Z.zinc_encrypt_batch(s.ctx, s.cache[COEFF], 7, m1, 1)           # bad form
    words = 2 * s.ctx.L * s.ctx.n
    misaligned = torch.empty((words + 1,), dtype=torch.uint64, device="cuda")[1:]
    with pytest.raises(Z.ZincError):
        Z.zinc_encrypt_batch(s.ctx, s.cache[COEFF], COEFF, m1, 1, out=misaligned)


def test_host_buffer_api_matches_device_api(Z, orc):
    s = setup_for(Z, orc, "C1")
    z = slots_batch(s.cfg, 0, 50)
    pt_h = torch.from_numpy(z).pin_memory()
    ct_h = torch.empty((50, 2, s.ctx.L, s.ctx.n), dtype=torch.uint64).pin_memory()
    Z.zinc_encrypt_batch_host(s.ctx, 0, s.cache[COEFF], COEFF, pt_h, 5, 0, ct_h, chunk=16)
    dev = Z.zinc_encrypt_batch(s.ctx, s.cache[COEFF], COEFF, torch.from_numpy(z).cuda(), 5, 0)
    assert torch.equal(ct_h, dev.cpu())
    Z.zinc_encrypt_batch_host(s.ctx, 1, s.pk, NTT, pt_h, 5, 0, ct_h, chunk=7)
    dev = Z.ckks_encrypt_batch(s.ctx, s.pk, NTT, torch.from_numpy(z).cuda(), 5, 0)
    assert torch.equal(ct_h, dev.cpu())


@pytest.mark.parametrize("path", ["zinc", "vanilla"])
def test_full_size_c3_bench_launch_sampled(Z, orc, path):
    """BASELINE C3 at full size (16384 messages, the bench's launch configuration):
    sampled messages bit-exact against the oracle, from int64 plaintexts."""
    s = setup_for(Z, orc, "C3")
    B = s.cfg.batch
    rng = np.random.default_rng(9)
    m_d = torch.randint(-(1 << 45), 1 << 45, (B, s.ctx.n), dtype=torch.int64, device="cuda",
                        generator=torch.Generator(device="cuda").manual_seed(9))
    seed = s.cfg.enc_seed
    if path == "zinc":
        ct = Z.zinc_encrypt_batch(s.ctx, s.cache[COEFF], COEFF, m_d, seed, 0)
    else:
        ct = Z.ckks_encrypt_batch(s.ctx, s.pk, NTT, m_d, seed, 0)
    torch.cuda.synchronize()
    idx = sorted(set([0, B - 1] + rng.integers(0, B, 4).tolist()))
    form = COEFF if path == "zinc" else NTT
    m = {b: m_d[b].cpu().numpy() for b in idx}
    got = {b: ct[b].cpu().numpy() for b in idx}
    del ct
    torch.cuda.empty_cache()
    key = s.o_pk if path == "vanilla" else orc.precompute_cache(s.P, s.o_pk, s.cfg.cache_seed, form)
    for b in idx:
        if path == "vanilla":
            want = orc.vanilla_encrypt(s.P, key, m[b], seed, b, form)
        else:
            want = orc.zinc_encrypt(s.P, key, form, m[b], seed, b)
        assert np.array_equal(got[b], want), b


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_int_peak_kernel_runs(Z, orc, variant):
    s = setup_for(Z, orc, "C3")
    sink = torch.zeros(2, dtype=torch.uint64, device="cuda")
    bf = Z.zinc_int_peak(s.ctx, 148 * 4, 100, sink, variant=variant)
    torch.cuda.synchronize()
    assert bf == 148 * 4 * 256 * 8 * 100
    with pytest.raises(Z.ZincError):
        Z.zinc_int_peak(s.ctx, 1, 1, sink, variant=4)


@pytest.mark.parametrize("knobs", [
    {0: 1, 1: 1 << 20, 2: 1},                 # 8-message chunks, PDL chain over 9 chunks
    {0: 7, 1: 3 << 20, 2: 0, 3: 0},           # plain stream order, no prefetch
    {0: 2, 1: 1 << 20, 3: 0},
    {4: 7},                                   # transform paths: 7-message chunks, PDL chain
    {4: 5, 2: 0},                             # transform paths: 5-message chunks, stream order
    {4: 1},                                   # one message per chunk
    {7: 0},                                   # Zinc COEFF plaintexts in double-buffered scratch
    {7: 2, 1: 1 << 20},                       # ... in the ciphertext slab, over 9 chunks
    {9: 0},                                   # transform paths: scratch plaintexts in natural order
    {9: 0, 4: 7},
])
def test_tuning_knobs_never_change_results(Z, orc, knobs):
    """Launch geometry (messages per CTA, encode chunk sizes, programmatic dependent launch,
    L2 prefetch) changes timing only: ciphertexts stay bit-identical to the default
    configuration, across chains of many chunks (the double-buffered scratch is reused)."""
    s = setup_for(Z, orc, "C3")
    z = torch.from_numpy(slots_batch(s.cfg, 0, 70)).cuda()
    calls = [lambda: Z.zinc_encrypt_batch(s.ctx, s.cache[COEFF], COEFF, z, 3, 10),
             lambda: Z.zinc_encrypt_batch(s.ctx, s.cache[NTT], NTT, z[:23], 3, 10),
             lambda: Z.ckks_encrypt_batch(s.ctx, s.pk, NTT, z[:17], 3, 10),
             lambda: Z.ckks_encrypt_batch(s.ctx, s.pk, COEFF, z[:11], 3, 10)]
    ref = [f() for f in calls]
    old = {k: Z.tune(k, v) for k, v in knobs.items()}
    try:
        got = [f() for f in calls]
        torch.cuda.synchronize()
    finally:
        for k, v in old.items():
            Z.tune(k, v)
    for a, b in zip(ref, got):
        assert torch.equal(a, b)


def test_c4_complex_slot_chain_bit_exact(Z, orc):
    """C4 complex slots (2-CTA cluster encode at N = 2^15) through a multi-chunk chain:
    2-message encode chunks, PDL on and off, equal to one another and to the oracle's
    encryption of the GPU-encoded plaintexts (first, middle and last chunk)."""
    s = setup_for(Z, orc, "C4")
    z = slots_batch(s.cfg, 0, 9)
    zz = torch.from_numpy(np.ascontiguousarray(np.stack([z.real, z.imag], axis=-1))).cuda()
    m = np64(Z.ckks_encode_batch(s.ctx, zz))
    outs = []
    for pdl in (1, 0):
        old = {k: Z.tune(k, v) for k, v in {Z.TUNE_ENCODE_CHUNK_BYTES: 2 * s.cfg.n * 8, Z.TUNE_PDL: pdl}.items()}
        try:
            outs.append(Z.zinc_encrypt_batch(s.ctx, s.cache[COEFF], COEFF, zz, 21, 300))
            torch.cuda.synchronize()
        finally:
            for k, v in old.items():
                Z.tune(k, v)
    assert torch.equal(outs[0], outs[1])
    _check_msgs(orc, s, "zinc", COEFF, m, np64(outs[0]), 21, 300, [0, 1, 4, 8])


def _full_size_slots_check(Z, orc, path, form, idx_fn):
    """Full C3 (16384 messages x 8192 slots, the A13 mix) from slots with the default
    launch configuration (the bench's timed call): sampled messages of the first, middle
    and last chunks bit-exact against the oracle's encryption of the GPU-encoded m."""
    s = setup_for(Z, orc, "C3")
    cfg = s.cfg
    B = cfg.batch
    z = slots_batch(cfg, 0, B)
    zd = torch.from_numpy(np.ascontiguousarray(z)).cuda()
    seed = cfg.enc_seed
    if path == "zinc":
        ct = Z.zinc_encrypt_batch(s.ctx, s.cache[form], form, zd, seed, 0)
    else:
        ct = Z.ckks_encrypt_batch(s.ctx, s.pk, form, zd, seed, 0)
    torch.cuda.synchronize()
    idx = idx_fn(B)
    got = {b: ct[b].cpu().numpy() for b in idx}
    m = np64(Z.ckks_encode_batch(s.ctx, zd[idx].contiguous()))
    del ct, zd
    torch.cuda.empty_cache()
    key = s.o_pk if path == "vanilla" else orc.precompute_cache(s.P, s.o_pk, cfg.cache_seed, form)
    for k, b in enumerate(idx):
        if path == "vanilla":
            want = orc.vanilla_encrypt(s.P, key, m[k], seed, b, form)
        else:
            want = orc.zinc_encrypt(s.P, key, form, m[k], seed, b)
        assert np.array_equal(got[b], want), (path, form, b)


def test_full_size_c3_slots_zinc_coeff_every_region(Z, orc):
    """The headline timed path: Zinc COEFF from slots, 64 PDL-chained 256-message chunks."""
    chunk = 256
    _full_size_slots_check(Z, orc, "zinc", COEFF, lambda B: [0, 1, chunk - 1, chunk, 31 * chunk + 7, 32 * chunk,
                                                             B // 2 - 1, B // 2, B - chunk, B - 2, B - 1])


@pytest.mark.parametrize("path,form", [("zinc", NTT), ("vanilla", NTT), ("vanilla", COEFF)])
def test_full_size_c3_slots_transform_paths(Z, orc, path, form):
    """Zinc NTT form and vanilla (both forms) from slots at full C3: chunks of 16 waves
    (4736 messages on 148 SMs), sampled in the first, middle and last chunk."""
    _full_size_slots_check(Z, orc, path, form, lambda B: [0, 4735, 4736, 8191, 9472, B - 1])


@pytest.mark.parametrize("name", ["C1", "C3", "C4"])
def test_ct_add_and_sum_bit_exact_and_decrypt(Z, orc, name):
    """Eq. 2 kernels: batched (+) and aggregation bit-exact against
    the oracle; the aggregate of k Zinc ciphertexts decrypts to the sum of the slots."""
    s = setup_for(Z, orc, name)
    cfg = s.cfg
    k = 7
    z = slots_batch(cfg, 0, k)
    zc = np.stack([z.real, z.imag], axis=-1) if cfg.complex_slots else z
    cts = Z.zinc_encrypt_batch(s.ctx, s.cache[COEFF], COEFF, torch.from_numpy(np.ascontiguousarray(zc)).cuda(), 9, 0)
    a, b = cts[:3].contiguous(), cts[3:6].contiguous()
    got_add = Z.zinc_ct_add_batch(s.ctx, a, b)
    assert np.array_equal(got_add.cpu().numpy(), orc.ct_add(s.P, a.cpu().numpy(), b.cpu().numpy()))
    tot = Z.zinc_ct_sum_batch(s.ctx, cts)
    assert np.array_equal(tot.cpu().numpy(), orc.ct_sum(s.P, cts.cpu().numpy()))
    assert not Z.zinc_ct_sum_batch(s.ctx, cts[:0]).cpu().numpy().any()        # empty batch -> zero
    _, st, zz = Z.ckks_decrypt_batch(s.ctx, s.sk, COEFF, tot[None].contiguous())
    assert int(st.sum()) == 0
    assert np.max(np.abs(zz[0].cpu().numpy() - z.sum(axis=0))) < k * cfg.tolerance()


def _setup_real15(Z, orc):
    """N = 2^15 with C4's primes but real slots (C4 itself has complex slots): the cluster
    encode's N = 2^15 instantiation."""
    from workloads import _cfg
    if "C4r" not in _setups:
        _setups["C4r"] = Setup(Z, orc, _cfg("C4r", 14, 15, [55] * 16, 40, 64, "uniform"))
    return _setups["C4r"]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4r"])
def test_small_cluster_path_bit_identical(Z, orc, name):
    """The small-batch latency path (k_small.cu): one message's encode over an 8-CTA cluster,
    and the Zinc COEFF form fused into the same launch with R cluster replicas per message.
    Plaintexts and ciphertexts are bit-identical to the throughput kernels (knob off) at every
    batch the path takes (1 .. SMs / 8) and at the first batch it does not, and the Zinc
    ciphertexts equal the oracle's encryption of those plaintexts."""
    s = _setup_real15(Z, orc) if name == "C4r" else setup_for(Z, orc, name)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    seed, base = 17, 900
    for B in sorted({1, 2, 3, 7, sms // 8, sms // 8 + 1}):
        z = torch.from_numpy(np.ascontiguousarray(slots_batch(s.cfg, 5, B))).cuda()
        calls = [lambda: Z.ckks_encode_batch(s.ctx, z),
                 lambda: Z.zinc_encrypt_batch(s.ctx, s.cache[COEFF], COEFF, z, seed, base),
                 lambda: Z.zinc_encrypt_batch(s.ctx, s.cache[NTT], NTT, z, seed, base),
                 lambda: Z.ckks_encrypt_batch(s.ctx, s.pk, NTT, z, seed, base)]
        got = [f() for f in calls]
        old = Z.tune(Z.TUNE_SMALL_CLUSTER, 0)
        try:
            ref = [f() for f in calls]
            torch.cuda.synchronize()
        finally:
            Z.tune(Z.TUNE_SMALL_CLUSTER, old)
        for k, (a, b) in enumerate(zip(got, ref)):
            assert torch.equal(a, b), (name, B, k)
        m = np64(got[0])
        idx = sorted({0, B // 2, B - 1})
        _check_msgs(orc, s, "zinc", COEFF, m, np64(got[1]), seed, base, idx)
        if name != "C4r":
            for b in idx:
                assert np.max(np.abs(m[b] - orc.encode(np64(z)[b], s.cfg.log_n, s.cfg.log_scale))) <= 1


@pytest.mark.parametrize("name,B", [("C3", 40), ("C4", 6)])
@pytest.mark.parametrize("split", [0, 1, 2])
def test_deinterleaved_scratch_plaintexts_bit_identical(Z, orc, name, B, split):
    """Slots feeding the NTT-form transform paths at N >= 2^14: the encode writes its scratch
    plaintexts de-interleaved by the path kernel's cluster size (TUNE_M_DEINT, default) or in
    natural order; same ciphertexts for every kernel family (TUNE_SPLIT), real and complex slots,
    over a multi-chunk chain, and equal to the oracle's encryption of the GPU-encoded plaintexts."""
    s = setup_for(Z, orc, name)
    z = slots_batch(s.cfg, 0, B)
    if s.cfg.complex_slots:
        z = np.stack([z.real, z.imag], axis=-1)
    zd = torch.from_numpy(np.ascontiguousarray(z)).cuda()
    m = np64(Z.ckks_encode_batch(s.ctx, zd))
    outs = {}
    for deint in (1, 0):
        old = {k: Z.tune(k, v) for k, v in {Z.TUNE_M_DEINT: deint, Z.TUNE_SPLIT: split, Z.TUNE_NTT_CHUNK_MSGS: 25}.items()}
        try:
            outs[deint] = (Z.zinc_encrypt_batch(s.ctx, s.cache[NTT], NTT, zd, 5, 77),
                           Z.ckks_encrypt_batch(s.ctx, s.pk, NTT, zd, 5, 77))
            torch.cuda.synchronize()
        finally:
            for k, v in old.items():
                Z.tune(k, v)
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)
    idx = [0, B // 2, B - 1]
    _check_msgs(orc, s, "zinc", NTT, m, np64(outs[1][0]), 5, 77, idx)
    _check_msgs(orc, s, "vanilla", NTT, m, np64(outs[1][1]), 5, 77, idx)
