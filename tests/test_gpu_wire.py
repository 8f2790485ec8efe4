"""PirServer.handle_frame on the GPU: reference-encoded request frames in,
reply frames byte-identical to the reference encoder's out (fast fixed-width
path and the generic fallback), plus the error mapping (server.py:128-208)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["desk_reduced", "toy", "q16", "ragged"])
def test_handle_frame_bytes_match_reference(golden, name):
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import wire
    from paper_2603_09190_b200.server import PirServer
    g = golden(name)
    fx = dict(np.load(os.path.join(GOLDEN, f"wire_{name}.npz")))
    ph = fx["params_hash"].tobytes()
    srv = PirServer(g.params(z), g.db)
    try:
        pf = lambda t, b: wire.pack_frame(t, ph, b)
        q = pf(wire.MSG_QUERY, fx["query_sep"].tobytes())[4:]
        # unknown client -> ERR_STATE
        r = srv.handle_frame(q)
        assert r[5] == wire.MSG_ERROR and int.from_bytes(r[38:42], "little") == wire.ERR_STATE
        assert srv.handle_frame(pf(wire.MSG_HINT_REQUEST, fx["hint_request"].tobytes())[4:]) == \
            pf(wire.MSG_ACK, b"")
        srv.wait_for_hints(timeout=120)
        want_sep = pf(wire.MSG_RESPONSE_SEPARATE, fx["resp_sep"].tobytes())
        want_comb = pf(wire.MSG_RESPONSE_COMBINED, fx["resp_comb"].tobytes())
        for _ in range(2):                       # graph capture, then replay
            assert srv.handle_frame(q) == want_sep
            assert srv.handle_frame(pf(wire.MSG_QUERY, fx["query_comb"].tobytes())[4:]) == want_comb
        assert srv.handle_frame(pf(wire.MSG_QUERY, fx["query_sep_minimal"].tobytes())[4:]) == want_sep
        # a reference Frame-like object works too
        fr = wire.unpack_frame(q)
        assert srv.handle_frame(fr) == want_sep
        # hint transfer: the stored k, then single-use -> ERR_INPUT (ValueError)
        cid = fx["client_id"].tobytes()
        ht = pf(wire.MSG_HINT_TRANSFER, cid + (0).to_bytes(8, "little"))[4:]
        k_body = fx["resp_comb"].tobytes()[:8] + wire.ints_field_rows(
            g.ints("k"), wire.WireLayout(g.params(z)).m2_bytes).tobytes()
        assert srv.handle_frame(ht) == pf(wire.MSG_HINT_TRANSFER_REPLY, k_body)
        r = srv.handle_frame(ht)
        assert r[5] == wire.MSG_ERROR and int.from_bytes(r[38:42], "little") == wire.ERR_INPUT
        # wrong parameter hash / unknown type -> ERR_PROTOCOL
        r = srv.handle_frame(wire.pack_frame(wire.MSG_QUERY, b"\x00" * 32, b"")[4:])
        assert int.from_bytes(r[38:42], "little") == wire.ERR_PROTOCOL
        r = srv.handle_frame(pf(77, b"")[4:])
        assert int.from_bytes(r[38:42], "little") == wire.ERR_PROTOCOL
        # unfresh query index -> HINT_PENDING
        far = fx["query_sep"].tobytes()
        far = far[:32] + (1000).to_bytes(8, "little") + far[40:]
        assert srv.handle_frame(pf(wire.MSG_QUERY, far)[4:]) == pf(wire.MSG_HINT_PENDING, b"")
    finally:
        srv.close()


def test_tcp_loopback_round_trip(golden):
    """A real TCP loopback server (127.0.0.1, as the reference's test_service)."""
    import socket
    import struct
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import wire
    from paper_2603_09190_b200.server import PirServer, serve, _read_exact
    g = golden("desk_reduced")
    fx = dict(np.load(os.path.join(GOLDEN, "wire_desk_reduced.npz")))
    ph = fx["params_hash"].tobytes()
    pir = PirServer(g.params(z), g.db)
    srv = serve(pir, "127.0.0.1", 0)
    try:
        with socket.create_connection(srv.server_address, timeout=60) as s:
            def rpc(t, body):
                s.sendall(wire.pack_frame(t, ph, body))
                (n,) = struct.unpack("<I", _read_exact(s, 4))
                return wire.unpack_frame(_read_exact(s, n))
            assert rpc(wire.MSG_HINT_REQUEST, fx["hint_request"].tobytes()).msg_type == wire.MSG_ACK
            pir.wait_for_hints(timeout=120)
            r = rpc(wire.MSG_QUERY, fx["query_sep"].tobytes())
            assert r.msg_type == wire.MSG_RESPONSE_SEPARATE and bytes(r.body) == fx["resp_sep"].tobytes()
            r = rpc(wire.MSG_QUERY, fx["query_comb"].tobytes())
            assert r.msg_type == wire.MSG_RESPONSE_COMBINED and bytes(r.body) == fx["resp_comb"].tobytes()
    finally:
        srv.shutdown()
        srv.server_close()
        pir.close()


@pytest.mark.parametrize("name", ["desk_reduced", "ragged", "uniform_key"])
def test_respond_batch_wire_matches_single(golden, name):
    """respond_batch_wire (configs[3]'s batch on wire fields, no Python ints):
    every query's limb rows equal respond_wire's, in both modes, with ck_o
    fields of mixed widths (the minimal-width encoding included), and the
    golden t / K for the golden query."""
    import random
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200.bigint import ints_to_limbs, limbs_to_ints
    g = golden(name)
    st = z.ServerGlobalState(g.params(z), g.db)
    pk = z.PaillierPublicKey(g.m, g.m.bit_length())
    reg = z.ClientRegistration(pk, g.seed, z.client_id_of(pk))
    reg.hints[0] = z.hint(st, reg, 0)
    lm = -(-g.m.bit_length() // 1024) * 32
    r = random.Random(17)
    rng = np.random.default_rng(17)
    cks, qus, modes = [], [], []
    for i in range(37):                       # > BATCH_SUB: several sub-batches
        ck = g.ints("ck_o") if i == 0 else [r.randrange(g.m) for _ in range(g.lwe["n"])]
        b = ints_to_limbs(ck, lm).view(np.uint8).reshape(len(ck), 4 * lm)
        w = 4 * lm if i % 3 else (max(v.bit_length() for v in ck) + 7) // 8
        cks.append(np.ascontiguousarray(b[:, :w]))
        qus.append(g.arr["qu0"] if i == 0 else rng.integers(0, g.lwe["q"], g.d0, dtype=np.uint64))
        modes.append(z.COMBINED if i % 4 == 1 else z.SEPARATE)
    modes[0] = z.SEPARATE
    modes[1] = z.COMBINED
    cks[1], qus[1] = cks[0], qus[0]
    out = z.respond_batch_wire(st, [reg] * 37, [0] * 37, modes, cks, qus)
    out = [o.copy() for o in out]
    assert limbs_to_ints(out[0]) == g.ints("t")
    assert limbs_to_ints(out[1]) == g.ints("K")
    for i in range(37):
        one = z.respond_wire(st, reg, 0, modes[i], cks[i], qus[i])
        assert np.array_equal(out[i], one), i
    with pytest.raises(KeyError):
        z.respond_batch_wire(st, [reg], [5], [z.SEPARATE], cks[:1], qus[:1])
    with pytest.raises(ValueError):
        z.respond_batch_wire(st, [reg], [0], [z.SEPARATE], [cks[0][:-1]], qus[:1])
