"""Host-side cost breakdown of PirServer.handle_frame at BASELINE configs[1]."""
import random
import statistics
import time

import numpy as np
import torch

import paper_2603_09190_b200 as z
from paper_2603_09190_b200 import _lib, build, wire, protocol
from paper_2603_09190_b200.server import PirServer
import bench

build.build()
_lib.load()
D0 = D1 = 32768
params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), D0, D1, 2048)
db = bench.db_slice(0, D1)
st = z.ServerGlobalState(params, db)
m = bench.paillier_modulus(2048, 2048)
pk = z.PaillierPublicKey(m, m.bit_length())
reg = z.ClientRegistration(pk, b"\x05" * 16, z.client_id_of(pk))
reg.hints[0] = z.hint(st, reg, 0)
rng = np.random.default_rng(1)
qu = rng.integers(0, 1 << 32, D0, dtype=np.uint64)
r = random.Random(2)
ck_o = [r.randrange(m) for _ in range(1024)]
srv = PirServer(params, None, state=st, hint_workers=1)
srv.close()
srv.registrations[reg.client_id] = reg
wl = wire.WireLayout(params)
body = wire.encode_query(wl, reg.client_id, 0, 0, ck_o, qu)
frame = wire.pack_frame(wire.MSG_QUERY, params.params_hash(), body)[4:]


def t(fn, n=50):
    for _ in range(3):
        fn()
    xs = []
    for _ in range(n):
        a = time.perf_counter()
        fn()
        xs.append(time.perf_counter() - a)
    return statistics.median(xs) * 1e6


dec = wire.decode_query(wl, body)
print("decode_query us", t(lambda: wire.decode_query(wl, body)))
print("respond_wire us", t(lambda: protocol.respond_wire(st, reg, 0, z.SEPARATE, dec[3], dec[4])))
limbs = protocol.respond_wire(st, reg, 0, z.SEPARATE, dec[3], dec[4])
print("field_rows us", t(lambda: wire.field_rows(limbs, wl.m_bytes)))
f = wire.field_rows(limbs, wl.m_bytes)
kf = srv._k_fields(reg.hints[0], wl.m2_bytes)
print("encode_sep us", t(lambda: wire.encode_response_separate(0, f, kf)))
b2 = wire.encode_response_separate(0, f, kf)
print("pack_frame us", t(lambda: wire.pack_frame(3, params.params_hash(), b2)))
print("handle_frame us", t(lambda: srv.handle_frame(frame)))
q = z.QueryMessage(reg.client_id, 0, z.SEPARATE, ck_o, qu)
print("respond us", t(lambda: z.respond(st, reg, q)))
print("params_hash us", t(lambda: params.params_hash()))
