"""B200-native ZipPIR server hot path (drop-in for the reference's
protocol.ServerGlobalState / hint / respond and PirServer.update_database).

Python host code over hand-written sm_100a CUDA kernels behind the C ABI in
include/zippir_b200.h (libzpir_b200.so, loaded by _lib.py). See DESIGN.md.
"""

from .params import LweParams, ProtocolParams, BINARY, UNIFORM, STANDARD, QUARTER_DELTA  # noqa: F401
from .paillier import (PaillierPublicKey, PaillierCiphertext, InvalidCiphertext,  # noqa: F401
                       multiexp, paillier_matmul, sample_ciphertext, trivial_encrypt, add,
                       add_batch)
from .protocol import (SEPARATE, COMBINED, ServerGlobalState, ClientHint,  # noqa: F401
                       ClientRegistration, QueryMessage, ResponseMessage, HintRequest,
                       client_id_of, derive_ck_r, hint, hints, respond, respond_batch,
                       respond_wire, respond_batch_wire, answer_wire,
                       refresh_hint, refresh_hints)

__all__ = [
    "LweParams", "ProtocolParams", "PaillierPublicKey", "PaillierCiphertext", "multiexp",
    "paillier_matmul", "sample_ciphertext", "ServerGlobalState", "ClientHint",
    "ClientRegistration", "QueryMessage", "ResponseMessage", "client_id_of", "derive_ck_r",
    "hint", "hints", "respond", "respond_batch", "respond_wire", "respond_batch_wire",
    "answer_wire", "refresh_hint", "refresh_hints", "SEPARATE", "COMBINED",
]
