"""Wire codec (paper_2603_09190_b200/wire.py) against bodies produced by the
reference's own encoder (tests/golden/wire_*.npz, made by make_golden.py).
CPU only: decode of both the fixed-width fast path and the generic fallback,
encode of response bodies from limb rows."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

CASES = ["desk_reduced", "toy", "q16", "ragged"]


def _fx(name):
    return dict(np.load(os.path.join(GOLDEN, f"wire_{name}.npz")))


@pytest.fixture(scope="module")
def w():
    from paper_2603_09190_b200 import wire
    return wire


@pytest.mark.parametrize("name", CASES)
def test_decode_query_fast_path_and_fallback(w, golden, name):
    import paper_2603_09190_b200 as z
    g = golden(name)
    fx = _fx(name)
    lay = w.WireLayout(g.params(z))
    body = fx["query_sep"].tobytes()
    assert len(body) == lay.query_body
    cid, qi, mode_b, ck, qu = w.decode_query(lay, body)
    assert cid == fx["client_id"].tobytes() and qi == 0 and mode_b == 0
    assert isinstance(ck, np.ndarray) and ck.shape == (g.lwe["n"], lay.m_bytes)
    assert [int.from_bytes(r.tobytes(), "little") for r in ck] == g.ints("ck_o")
    assert np.array_equal(qu.astype(np.uint64), g.arr["qu0"])
    assert w.decode_query(lay, fx["query_comb"].tobytes())[2] == 1
    # minimal-width integers (generic decoder unless every field happens to
    # have full width): same values
    cid2, qi2, m2, ck2, qu2 = w.decode_query(lay, fx["query_sep_minimal"].tobytes())
    if isinstance(ck2, np.ndarray):
        ck2 = [int.from_bytes(r.tobytes(), "little") for r in ck2]
    assert cid2 == cid and ck2 == g.ints("ck_o") and [int(x) for x in qu2] == \
        [int(x) for x in g.arr["qu0"]]


@pytest.mark.parametrize("name", CASES)
def test_encode_responses_from_limbs(w, golden, name):
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200.bigint import ints_to_limbs
    g = golden(name)
    fx = _fx(name)
    lay = w.WireLayout(g.params(z))
    L = -(-lay.m_bytes // 4)
    t = w.field_rows(ints_to_limbs(g.ints("t"), L + 1), lay.m_bytes)     # wider limb rows
    k = w.ints_field_rows(g.ints("k"), lay.m2_bytes)
    assert w.encode_response_separate(0, t, k) == fx["resp_sep"].tobytes()
    K = w.field_rows(ints_to_limbs(g.ints("K"), 2 * L), lay.m2_bytes)
    assert w.encode_response_combined(0, K) == fx["resp_comb"].tobytes()
    qi, tt, kk = w.decode_response(lay, fx["resp_sep"].tobytes(), combined=False)
    assert tt == g.ints("t") and kk == g.ints("k")


def test_frames_and_errors(w, golden):
    import paper_2603_09190_b200 as z
    g = golden("desk_reduced")
    fx = _fx("desk_reduced")
    ph = fx["params_hash"].tobytes()
    assert ph == g.params(z).params_hash()
    f = w.pack_frame(w.MSG_QUERY, ph, fx["query_sep"].tobytes())
    fr = w.unpack_frame(f[4:])
    assert fr.msg_type == w.MSG_QUERY and fr.params_hash == ph
    assert int.from_bytes(f[:4], "little") == len(f) - 4
    with pytest.raises(w.WireError):
        w.unpack_frame(b"\x02" + f[5:])
    lay = w.WireLayout(g.params(z))
    with pytest.raises(ValueError):
        w.decode_query(lay, fx["query_sep"].tobytes()[:-1])
    with pytest.raises(w.WireError):
        w.decode_query(lay, fx["query_sep"].tobytes() + b"\x00")
    m, seed = w.decode_hint_request(lay, fx["hint_request"].tobytes())
    assert m == g.m and seed == g.seed
    with pytest.raises(ValueError):
        w.field_rows(np.full((1, 2), 0xFFFFFFFF, dtype=np.uint32), 5)


def test_tcp_serve_loop_cpu(w):
    """The TCP loop frames requests and replies (a stand-in handler; CPU only)."""
    import socket
    import struct
    from paper_2603_09190_b200.server import serve, _read_exact

    class Echo:
        def handle_frame(self, payload):
            f = w.unpack_frame(payload)
            return w.pack_frame(w.MSG_ACK, f.params_hash, bytes(f.body[::-1]))

    srv = serve(Echo(), "127.0.0.1", 0)
    try:
        with socket.create_connection(srv.server_address, timeout=10) as s:
            for body in (b"", b"abc", bytes(range(256)) * 40):
                s.sendall(w.pack_frame(w.MSG_QUERY, b"\x07" * 32, body))
                (n,) = struct.unpack("<I", _read_exact(s, 4))
                f = w.unpack_frame(_read_exact(s, n))
                assert f.msg_type == w.MSG_ACK and bytes(f.body) == body[::-1]
    finally:
        srv.shutdown()
        srv.server_close()
