"""Generate golden fixtures by running the UNMODIFIED reference package.

Build-container only: imports /root/reference/pkg/src/zippir with the gmpy2
stand-in in tests/golden/_shim (gmpy2 is absent, there is no network). The
outputs (tests/golden/*.npz, *.json) are committed; nothing on the GPU box
reads /root/reference.

    python tests/golden/make_golden.py [--skip-tiny]

Each case records the reference's own outputs on seeded inputs:
  * ProtocolParams layout (gamma, capacity, d1'), public matrix A, global
    hint H = -db^T A mod q (protocol.py:91-95, :195-217)
  * one client (keygen from random.Random(seed)), derive_ck_r for qi=0,
    the hint entries k_g = multiexp(ck_r, H_scaled[g]) (protocol.py:285-296,
    paillier.py:134-208)
  * a query, b = db_matvec(qu0), respond() in SEPARATE and COMBINED mode,
    and extract() == db[i0] (protocol.py:299-396)
  * multiexp known-answer vectors (paillier.py:134-193) incl. the edge cases
    (all-zero exponents -> 1, maxbits <= 6 -> w = maxbits, single base)
"""

import argparse
import hashlib
import json
import os
import random
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, os.path.join(HERE, "_shim"))
sys.path.insert(0, REF_SRC)

from zippir import counters, paillier, protocol  # noqa: E402
from zippir.lwe import LweParams  # noqa: E402
from zippir.protocol import (COMBINED, SEPARATE, ClientRegistration,  # noqa: E402
                             ProtocolParams, ServerGlobalState, client_id_of,
                             derive_ck_r, extract, hint, query, respond, setup)


def le_bytes(values, width):
    """Python ints -> (len, width) uint8 little-endian rows."""
    buf = b"".join(int(v).to_bytes(width, "little") for v in values)
    return np.frombuffer(buf, dtype=np.uint8).reshape(len(values), width).copy()


def sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def protocol_case(name, lwe_kw, d0, d1, bits, seed, db=None, scale_regime=None,
                  i0=None, store_full=True):
    t_start = time.time()
    lwe = LweParams(**lwe_kw)
    kw = dict(lwe=lwe, d0=d0, d1=d1, paillier_bits=bits)
    if scale_regime:
        kw["scale_regime"] = scale_regime
    params = ProtocolParams(**kw)
    rng = random.Random(seed)
    if db is None:
        db = np.array([[rng.randrange(lwe.p) for _ in range(d1)]
                       for _ in range(d0)], dtype=np.int64)
    state = ServerGlobalState(params, db)
    client, hreq = setup(params, rng)
    reg = ClientRegistration(hreq.pk, hreq.seed, client_id_of(hreq.pk))
    qi = 0
    ck_r = derive_ck_r(reg.pk, reg.seed, qi, lwe.n)
    with counters.measure() as mh:
        h = hint(state, reg, qi)
    reg.hints[qi] = h
    if i0 is None:
        i0 = rng.randrange(d0)
    qmsg, secret = query(client, params, i0, qi, rng, mode=SEPARATE, A=state.A)
    b = state.db_matvec(qmsg.qu0)
    r_sep = respond(state, reg, qmsg, mode=SEPARATE)
    with counters.measure() as mc:
        r_comb = respond(state, reg, qmsg, mode=COMBINED)
    rec_sep = extract(client.sk_paillier, params, r_sep)
    rec_comb = extract(client.sk_paillier, params, r_comb)
    want = [int(x) for x in db[i0]]
    assert rec_sep == want and rec_comb == want, name

    m = reg.pk.m
    mb = (bits + 7) // 8
    H = np.array(state.H, dtype=np.uint64)
    meta = dict(
        name=name, lwe=lwe_kw, d0=d0, d1=d1, paillier_bits=bits,
        scale_regime=params.scale_regime, seed=seed,
        gamma=str(params.gamma), capacity=params.capacity,
        d1_prime=params.d1_prime, params_hash=params.params_hash().hex(),
        p=hex(client.sk_paillier.p), q=hex(client.sk_paillier.q), m=hex(m),
        client_seed=reg.seed.hex(), query_index=qi, i0=i0,
        A_sha256=sha(state.A.astype("<u8")), H_sha256=sha(H.astype("<u8")),
        db_sha256=sha(np.asarray(db, dtype=np.uint8)),
        hint_group_mults=mh.delta.group_mult,
        combined_adds=mc.delta.add, combined_modexp=mc.delta.modexp,
        ref_seconds=round(time.time() - t_start, 1),
    )
    arrays = dict(
        qu0=np.asarray(qmsg.qu0, dtype=np.uint64),
        ck_o=le_bytes(qmsg.ck_o, mb),
        b=np.asarray(b, dtype=np.uint64),
        t=le_bytes(r_sep.t, mb),
        k=le_bytes([c.c for c in h.entries], 2 * mb),
        K=le_bytes([c.c for c in r_comb.k], 2 * mb),
        ck_r=le_bytes([c.c for c in ck_r], 2 * mb),
        A_row0=np.asarray(state.A[0], dtype=np.uint64),
        H_rows=H[[0, d1 // 2, d1 - 1]],
        record=np.asarray(want, dtype=np.int64),
    )
    if store_full:
        arrays["db"] = np.asarray(db, dtype=np.uint8)
        arrays["H"] = H
        arrays["A"] = np.asarray(state.A, dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    with open(os.path.join(HERE, f"{name}.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(f"{name}: d1'={params.d1_prime} cap={params.capacity} "
          f"{meta['ref_seconds']} s", flush=True)


def multiexp_cases():
    out = []
    rng = random.Random(4242)
    for bits in (64, 768, 2048):
        _, sk = paillier.keygen(bits, random.Random(bits + 1))
        pk = sk.pk
        m2 = pk.m2

        def rnd_cts(k):
            return [paillier.PaillierCiphertext(rng.randrange(m2)) for _ in range(k)]
        cases = [
            ("random", rnd_cts(16), [rng.randrange(1 << 200) for _ in range(16)]),
            ("zero_exps", rnd_cts(4), [0, 0, 0, 0]),
            ("single", rnd_cts(1), [rng.randrange(1 << 64)]),
            ("small_w", rnd_cts(7), [rng.randrange(1 << 5) for _ in range(7)]),
            ("powers", rnd_cts(5), [1 << (7 * i) for i in range(5)]),
            ("one_hot", rnd_cts(9), [0] * 4 + [rng.randrange(1 << 300)] + [0] * 4),
            ("long", rnd_cts(33), [rng.randrange(1 << (bits - 32 if bits > 64 else 60))
                                   for _ in range(33)]),
        ]
        for tag, cts, exps in cases:
            r = paillier.multiexp(pk, cts, exps)
            out.append(dict(bits=bits, tag=tag, m=hex(pk.m),
                            bases=[hex(c.c) for c in cts],
                            exps=[hex(e) for e in exps], result=hex(r.c)))
    with open(os.path.join(HERE, "multiexp_kat.json"), "w") as f:
        json.dump(out, f, indent=0)
    print("multiexp_kat:", len(out), flush=True)


def prg_cases():
    """Stream / public_matrix / sample_ciphertext known answers (prg.py)."""
    from zippir.prg import Stream
    out = dict(
        stream_seed00_dom3_first64=Stream(b"\x00" * 16, 3).read(64).hex(),
        stream_seedab_dom1_idx=Stream(b"\xab" * 16, 1, (5 << 32) | 7).read(48).hex(),
        below=[Stream(bytes(range(16)), 4, i).below((1 << 100) + 12345) for i in range(8)],
    )
    out["below"] = [hex(x) for x in out["below"]]
    with open(os.path.join(HERE, "prg_kat.json"), "w") as f:
        json.dump(out, f, indent=1)


def wire_cases(names=("desk_reduced", "toy", "q16", "ragged")):
    """Reference wire bodies (wire.py:128-206) for the golden queries/answers:
    query bodies (both modes), response bodies, hint request, and a body with
    non-canonical widths that only the generic decoder accepts."""
    from zippir import wire
    from zippir.paillier import PaillierPublicKey
    for name in names:
        meta = json.load(open(os.path.join(HERE, f"{name}.json")))
        arr = np.load(os.path.join(HERE, f"{name}.npz"))
        ints = lambda k: [int.from_bytes(r.tobytes(), "little") for r in arr[k]]
        lw = meta["lwe"]
        kw = dict(lwe=LweParams(**lw), d0=meta["d0"], d1=meta["d1"],
                  paillier_bits=meta["paillier_bits"], scale_regime=meta["scale_regime"])
        params = ProtocolParams(**kw)
        lay = wire.Layout(params.paillier_bits, lw["n"], lw["q"].bit_length() - 1,
                          params.d0, params.d1_prime)
        m = int(meta["m"], 16)
        pk = PaillierPublicKey(m, m.bit_length())
        cid = client_id_of(pk)
        qu0 = [int(x) for x in arr["qu0"]]
        out = dict(
            params_hash=np.frombuffer(params.params_hash(), np.uint8),
            client_id=np.frombuffer(cid, np.uint8),
            hint_request=np.frombuffer(wire.encode_hint_request(
                lay, m, bytes.fromhex(meta["client_seed"])), np.uint8),
            query_sep=np.frombuffer(wire.encode_query(lay, cid, 0, 0, ints("ck_o"), qu0), np.uint8),
            query_comb=np.frombuffer(wire.encode_query(lay, cid, 0, 1, ints("ck_o"), qu0), np.uint8),
            resp_sep=np.frombuffer(wire.encode_response_separate(lay, 0, ints("t"), ints("k")),
                                   np.uint8),
            resp_comb=np.frombuffer(wire.encode_response_combined(lay, 0, ints("K")), np.uint8),
        )
        # minimal-width integers: valid for the reference's prefixed decoder
        from zippir.serial import encode_bigint
        import struct
        body = cid + struct.pack("<QB", 0, 0) + b"".join(encode_bigint(v) for v in ints("ck_o")) \
            + b"".join(encode_bigint(v) for v in qu0)
        assert wire.decode_query(lay, body)[3] == ints("ck_o")
        out["query_sep_minimal"] = np.frombuffer(body, np.uint8)
        np.savez_compressed(os.path.join(HERE, f"wire_{name}.npz"), **out)
    print("wire fixtures:", names, flush=True)


def dbfile_cases():
    """Reference-serialized database files (dbfile.py:24-31)."""
    from zippir import dbfile
    arr = np.load(os.path.join(HERE, "desk_reduced.npz"))
    db = dbfile.DatabaseFile(32, 48, 256, 48, arr["db"].astype(np.int64))
    dbfile.save(db, os.path.join(HERE, "desk_reduced.zpirdb"))
    f = dbfile.ingest(bytes(range(80)), 8, 20, p=16)   # two base-16 digits per byte
    dbfile.save(f, os.path.join(HERE, "ingest_p16.zpirdb"))
    print("dbfile fixtures", flush=True)


def gamma_cases():
    """Batch scales other than 2^32 (compress.py:36-43): uniform key with
    quarter-delta (gamma = q^2 = 2^64), standard regime (gamma = q + n q),
    and q < 2^32 (gamma = q = 2^16)."""
    protocol_case("uniform_key", dict(n=32, q=1 << 32, p=256, noise_sigma=6.4,
                                      key_dist="uniform"), 40, 70, 1024, seed=21)
    protocol_case("standard32", dict(n=16, q=1 << 32, p=256, noise_sigma=6.4,
                                     key_dist="binary"), 48, 90, 1024, seed=22,
                  scale_regime="standard")
    protocol_case("q16", dict(n=32, q=1 << 16, p=16, noise_sigma=1.0, key_dist="binary"),
                  64, 100, 1024, seed=23)


def compress_cases():
    """The reference's standalone compressor (compress.py:99-258) on seeded
    inputs: lwe_compress, fast_lwe_compress (expanded key), batched_lwe_compress
    and fast_batched_lwe_compress -> compress_kat.json."""
    from zippir import compress
    from zippir.lwe import LweCiphertext
    out = []
    for bits, n, q, key_dist, ncts, seed in ((768, 64, 1 << 32, "binary", 4, 31),
                                             (1024, 32, 1 << 16, "binary", 3, 32),
                                             (2048, 128, 1 << 32, "uniform", 2, 33)):
        rng = random.Random(seed)
        pk, sk = paillier.keygen(bits, rng)
        lwe = LweParams(n=n, q=q, p=256 if q > 256 else 16, noise_sigma=0.0, key_dist=key_dist)
        lwe_sk = [rng.randrange(2) if key_dist == "binary" else rng.randrange(q)
                  for _ in range(n)]
        ck = compress.make_compression_key(pk, lwe, lwe_sk, rng)
        cts = [LweCiphertext(np.array([rng.randrange(q) for _ in range(n)], dtype=np.uint64),
                             rng.randrange(q)) for _ in range(ncts)]
        single = [compress.lwe_compress(ck, ct).x.c for ct in cts]
        eck = compress.expand_compression_key(ck)
        fast = [compress.fast_lwe_compress(eck, ct).x.c for ct in cts]
        gamma = compress.select_scale(lwe)
        ell = min(len(cts), compress.batch_capacity(pk, gamma))
        batched = compress.batched_lwe_compress(ck, cts[:ell], gamma).x.c
        fast_batched = compress.fast_batched_lwe_compress(ck, cts[:ell], gamma).x.c
        out.append(dict(bits=bits, n=n, q=q, key_dist=key_dist, m=hex(pk.m),
                        ck=[hex(c.c) for c in ck.ck],
                        cts=[dict(a=[int(x) for x in ct.a], b=int(ct.b)) for ct in cts],
                        lwe_compress=[hex(v) for v in single],
                        fast_lwe_compress=[hex(v) for v in fast],
                        gamma=str(gamma), ell=ell, batched=hex(batched),
                        fast_batched=hex(fast_batched)))
    with open(os.path.join(HERE, "compress_kat.json"), "w") as f:
        json.dump(out, f, indent=0)
    print("compress_kat:", len(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-tiny", action="store_true")
    ap.add_argument("--wire-only", action="store_true", help="only the wire fixtures")
    ap.add_argument("--compress-only", action="store_true", help="only compress_kat.json")
    ap.add_argument("--gamma-only", action="store_true",
                    help="only the batch-scale cases (gamma != 2^32)")
    args = ap.parse_args()
    if args.compress_only:
        compress_cases()
        return
    if args.wire_only:
        wire_cases()
        dbfile_cases()
        return
    gamma_cases()
    if args.gamma_only:
        return
    prg_cases()
    multiexp_cases()
    compress_cases()
    # reference's toy fixture (tests/test_protocol.py:12-19): standard regime
    protocol_case("toy", dict(n=4, q=16, p=4, noise_sigma=0.0, key_dist="binary"),
                  4, 4, 64, seed=0xC0FFEE, scale_regime="standard")
    # reference's reduced desk (tests/test_protocol.py:190-209)
    protocol_case("desk_reduced", dict(n=64, q=1 << 32, p=256, noise_sigma=6.4,
                                       key_dist="binary"), 32, 48, 768, seed=11)
    # ragged shapes: d0 not a multiple of 16, d1 not a multiple of cap or 128
    protocol_case("ragged", dict(n=256, q=1 << 32, p=256, noise_sigma=6.4,
                                 key_dist="binary"), 777, 130, 1024, seed=12)
    # all-zero database
    protocol_case("zero_db", dict(n=64, q=1 << 32, p=256, noise_sigma=6.4,
                                  key_dist="binary"), 32, 48, 768, seed=13,
                  db=np.zeros((32, 48), dtype=np.int64))
    # all-255 database (max symbols: worst-case accumulator magnitudes)
    protocol_case("max_db", dict(n=128, q=1 << 32, p=256, noise_sigma=6.4,
                                 key_dist="binary"), 300, 200, 1024, seed=14,
                  db=np.full((300, 200), 255, dtype=np.int64))
    if not args.skip_tiny:
        # BASELINE.json configs[0]: 1024x1024, n=1024, 2048-bit, bench.py:167 DB
        d0 = d1 = 1024
        db = np.frombuffer(np.random.default_rng(7).bytes(d0 * d1),
                           dtype=np.uint8).reshape(d0, d1)
        protocol_case("tiny", dict(n=1024, q=1 << 32, p=256, noise_sigma=6.4,
                                   key_dist="binary"), d0, d1, 2048, seed=2048,
                      db=db, store_full=False)
    wire_cases()
    dbfile_cases()


if __name__ == "__main__":
    main()
