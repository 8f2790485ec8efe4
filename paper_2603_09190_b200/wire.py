"""Wire codec for the query / response frames, straight from device limbs
(SURVEY.md 8f rank 4).

Byte-compatible with the reference's frame format (wire.py:1-206,
serial.py:11-36): frame = u32-LE payload length, version u8, message type
u8, 32-byte parameter hash, body; body big integers are a u32-LE byte count
followed by the little-endian magnitude, padded to the parameter-determined
field width. The reference decodes every integer into a Python int and
encodes every result with int.to_bytes. Here a query body whose fields all
carry the fixed widths (what every conforming client sends,
wire.py:141-148) is read as two strided numpy views -- ck_o as (n, m_bytes)
byte rows that go straight into the device limb buffer, qu0 as (d0,) u32 --
and the response body is assembled from the device's limb rows with one
vectorised copy. Anything else (non-canonical widths) falls back to the
generic prefixed decoder, so every body the reference accepts is accepted.
"""

import struct

import numpy as np

WIRE_VERSION = 1
HEADER_BYTES = 1 + 1 + 32
FRAME_PREFIX_BYTES = 4

MSG_HINT_REQUEST = 1
MSG_QUERY = 2
MSG_RESPONSE_SEPARATE = 3
MSG_RESPONSE_COMBINED = 4
MSG_HINT_TRANSFER = 5
MSG_HINT_TRANSFER_REPLY = 6
MSG_ACK = 7
MSG_ERROR = 8
MSG_HINT_PENDING = 9

ERR_INPUT = 10
ERR_PROTOCOL = 20
ERR_STATE = 30
ERR_CRYPTO = 40

MODE_BY_BYTE = {0: "separate", 1: "combined"}   # server.py:25
BYTE_BY_MODE = {v: k for k, v in MODE_BY_BYTE.items()}


class WireError(Exception):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class Frame:
    __slots__ = ("msg_type", "params_hash", "body")

    def __init__(self, msg_type, params_hash, body):
        self.msg_type, self.params_hash, self.body = msg_type, params_hash, body


def pack_frame(msg_type: int, params_hash: bytes, body) -> bytes:
    if len(params_hash) != 32:
        raise WireError(ERR_INPUT, "params hash must be 32 bytes")
    n = HEADER_BYTES + len(body)
    return b"".join((struct.pack("<IBB", n, WIRE_VERSION, msg_type), params_hash, body))


def unpack_frame(data: bytes) -> Frame:
    """Payload (without the u32 length prefix) -> Frame."""
    if len(data) < HEADER_BYTES:
        raise WireError(ERR_PROTOCOL, "short frame")
    if data[0] != WIRE_VERSION:
        raise WireError(ERR_PROTOCOL, f"unsupported wire version {data[0]}")
    mv = memoryview(data)
    return Frame(data[1], bytes(mv[2:34]), mv[34:])   # body: zero-copy view


class WireLayout:
    """Field widths fixed by the parameters (wire.py:91-125)."""

    def __init__(self, params):
        lwe = params.lwe
        bits = params.paillier_bits
        self.m_bytes = (bits + 7) // 8
        self.m2_bytes = (2 * bits + 7) // 8
        self.q_bytes = (lwe.q.bit_length() - 1 + 7) // 8
        self.n = lwe.n
        self.d0 = params.d0
        d1p = getattr(params, "d1_prime", None)
        if d1p is None:
            from .params import capacity_of
            d1p = -(-params.d1 // capacity_of(params))
        self.d1_prime = d1p
        self.query_body = 32 + 9 + self.n * (4 + self.m_bytes) + self.d0 * (4 + self.q_bytes)


# -- query decode --------------------------------------------------------------

def _prefixed(buf: memoryview, off: int):
    if off + 4 > len(buf):
        raise ValueError("truncated big-integer field")
    (nb,) = struct.unpack_from("<I", buf, off)
    off += 4
    if off + nb > len(buf):
        raise ValueError("truncated big-integer field")
    return int.from_bytes(buf[off:off + nb], "little"), off + nb


def decode_query(lay: WireLayout, body):
    """-> (client_id, query_index, mode_byte, ck_o, qu0).

    Fast path: ck_o is an (n, m_bytes) uint8 view of the body and qu0 a
    (d0,) uint32 array (q_bytes <= 4). Fallback: Python-int lists exactly as
    the reference's decoder produces them (wire.py:151-166)."""
    mv = memoryview(body)
    if len(mv) < 32 + 9:
        raise WireError(ERR_INPUT, "bad query length")
    client_id = bytes(mv[:32])
    qi, mode_b = struct.unpack_from("<QB", mv, 32)
    if len(mv) == lay.query_body and lay.q_bytes <= 4:
        cw = 4 + lay.m_bytes
        ck = np.frombuffer(mv, dtype=np.uint8, count=lay.n * cw, offset=41).reshape(lay.n, cw)
        q0 = 41 + lay.n * cw
        if lay.q_bytes == 4:
            # (prefix, value) u32 pairs: one strided view, no copy
            qv = np.frombuffer(mv, dtype="<u4", count=2 * lay.d0, offset=q0)
            qpre, qu = qv[0::2], qv[1::2]
        else:
            qf = np.frombuffer(mv, dtype=np.uint8, offset=q0).reshape(lay.d0, 4 + lay.q_bytes)
            qpre = qf[:, :4].view("<u4")
            qb = np.zeros((lay.d0, 4), dtype=np.uint8)
            qb[:, : lay.q_bytes] = qf[:, 4:]
            qu = qb.view("<u4").reshape(lay.d0)
        if (ck[:, :4].view("<u4") == lay.m_bytes).all() and (qpre == lay.q_bytes).all():
            return client_id, qi, mode_b, ck[:, 4:], qu
    off = 41
    ck_o = []
    for _ in range(lay.n):
        v, off = _prefixed(mv, off)
        ck_o.append(v)
    qu0 = []
    for _ in range(lay.d0):
        v, off = _prefixed(mv, off)
        qu0.append(v)
    if off != len(mv):
        raise WireError(ERR_INPUT, "trailing bytes in query")
    return client_id, qi, mode_b, ck_o, qu0


def encode_query(lay: WireLayout, client_id: bytes, query_index: int, mode: int, ck_o, qu0) -> bytes:
    """Client-side encoder (wire.py:141-148), used by tests and the bench."""
    parts = [client_id, struct.pack("<QB", query_index, mode)]
    for v in ck_o:
        parts += [struct.pack("<I", lay.m_bytes), int(v).to_bytes(lay.m_bytes, "little")]
    for v in qu0:
        parts += [struct.pack("<I", lay.q_bytes), int(v).to_bytes(lay.q_bytes, "little")]
    return b"".join(parts)


# -- response encode from limb rows ------------------------------------------------

def field_rows(limbs: np.ndarray, width: int) -> np.ndarray:
    """(count, L) u32 limb rows -> (count, 4 + width) prefixed fixed-width fields."""
    limbs = np.ascontiguousarray(limbs, dtype="<u4")
    count = limbs.shape[0]
    raw = limbs.view(np.uint8).reshape(count, -1)
    out = np.zeros((count, 4 + width), dtype=np.uint8)
    out[:, :4] = np.frombuffer(struct.pack("<I", width), dtype=np.uint8)
    w = min(width, raw.shape[1])
    out[:, 4:4 + w] = raw[:, :w]
    if raw.shape[1] > width and raw[:, width:].any():
        raise ValueError("value wider than its wire field")
    return out


def ints_field_rows(values, width: int) -> np.ndarray:
    """Python ints -> prefixed fixed-width fields (serial.py:25-29)."""
    out = np.zeros((len(values), 4 + width), dtype=np.uint8)
    out[:, :4] = np.frombuffer(struct.pack("<I", width), dtype=np.uint8)
    for i, v in enumerate(values):
        if v < 0:
            raise ValueError("negative integers are not encodable")
        out[i, 4:] = np.frombuffer(int(v).to_bytes(width, "little"), dtype=np.uint8)
    return out


def encode_response_separate(query_index: int, t_fields: np.ndarray, k_fields: np.ndarray) -> bytes:
    """wire.py:169-173: qi, d1' t fields (m_bytes), d1' k fields (m2_bytes)."""
    return b"".join((struct.pack("<Q", query_index), t_fields, k_fields))


def encode_response_combined(query_index: int, K_fields: np.ndarray) -> bytes:
    """wire.py:190-193 (also the hint transfer reply, wire.py:219-223)."""
    return b"".join((struct.pack("<Q", query_index), K_fields))


def pack_reply(msg_type: int, params_hash: bytes, query_index: int, *fields) -> bytes:
    """pack_frame(msg_type, params_hash, encode_response_*(query_index, *fields))
    assembled in one pass (no intermediate body copy)."""
    n = HEADER_BYTES + 8 + sum(f.nbytes for f in fields)
    return b"".join((struct.pack("<IBB", n, WIRE_VERSION, msg_type), params_hash,
                     struct.pack("<Q", query_index), *fields))


def decode_response(lay: WireLayout, body: bytes, combined: bool):
    """Client-side decoder (wire.py:176-206) for tests: -> (qi, t, k) or (qi, K)."""
    mv = memoryview(body)
    (qi,) = struct.unpack_from("<Q", mv)
    off = 8
    lists = []
    for _ in range(1 if combined else 2):
        vals = []
        for _ in range(lay.d1_prime):
            v, off = _prefixed(mv, off)
            vals.append(v)
        lists.append(vals)
    if off != len(mv):
        raise WireError(ERR_INPUT, "trailing bytes in response")
    return (qi, *lists)


def encode_error(code: int, message: str) -> bytes:
    return struct.pack("<I", code) + message.encode()


def decode_hint_request(lay: WireLayout, body: bytes):
    """wire.py:133-138: g = m + 1 (prefixed), then the seed."""
    mv = memoryview(body)
    g, off = _prefixed(mv, 0)
    rest = bytes(mv[off:])
    if len(rest) != 16:
        raise WireError(ERR_INPUT, "bad hint request length")
    return g - 1, rest


def decode_hint_transfer(body: bytes):
    if len(body) != 40:
        raise WireError(ERR_INPUT, "bad hint transfer length")
    return bytes(body[:32]), struct.unpack("<Q", body[32:])[0]
