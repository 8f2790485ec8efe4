"""PirServer's reference constructor and its hint-store delegation, on CPU
(the device state is replaced by a stand-in; no GPU needed):

* PirServer(params, db, store_dir, basis) positional order (server.py:30-31);
* a store_dir string opens the reference's own HintStore when the reference
  package is importable (in this container: /root/reference with the gmpy2
  stand-in of tests/golden/_shim), registrations are saved and restored;
* a duck-typed store object is used as is;
* the slot decomposition is kept only for each client's look-ahead window.
"""

import os
import sys
from types import SimpleNamespace

import pytest

from paper_2603_09190_b200 import server
from paper_2603_09190_b200.paillier import PaillierPublicKey

REF_SRC = "/root/reference/pkg/src"
SHIM = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "_shim")


def _params():
    return SimpleNamespace(hints_per_client=2, paillier_bits=64)


class MemStore:
    def __init__(self):
        self.regs, self.hints, self.purged = {}, {}, []

    def save_registration(self, cid, pk, seed):
        self.regs[cid] = (pk, seed)

    def load_registrations(self):
        for cid, (pk, seed) in self.regs.items():
            yield cid, pk, seed

    def save_hint(self, cid, qi, version, entries):
        self.hints[(cid, qi, version)] = list(entries)

    def load_hints(self, cid, version):
        return {qi: e for (c, qi, v), e in self.hints.items() if c == cid and v == version}

    def purge_stale(self, cid, version):
        self.purged.append((cid, version))


def _server(store_dir=None, store=None):
    state = SimpleNamespace(db_version=0, device="cpu")
    return server.PirServer(_params(), None, store_dir, None, store=store, state=state,
                            hint_workers=0)


def test_duck_typed_store_and_restore():
    st = MemStore()
    pk = PaillierPublicKey((1 << 63) + 29, 64)
    st.regs[b"c1"] = (pk, b"\x01" * 16)
    st.hints[(b"c1", 0, 0)] = [5, 6]
    srv = _server(store=st)
    try:
        reg = srv.registrations[b"c1"]
        assert [c.c for c in reg.hints[0].entries] == [5, 6]
        assert reg.hints[0].db_version == 0
        assert srv.jobs.qsize() >= 1          # the missing look-ahead hint was queued
    finally:
        srv.close()
    srv2 = _server(store_dir=st)             # an object passed positionally as store_dir
    try:
        assert b"c1" in srv2.registrations
        cid = srv2.register(PaillierPublicKey((1 << 63) + 123, 64), b"\x02" * 16)
        assert cid in st.regs
    finally:
        srv2.close()


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present")
def test_store_dir_string_opens_reference_hintstore(tmp_path, monkeypatch):
    monkeypatch.syspath_prepend(REF_SRC)
    monkeypatch.syspath_prepend(SHIM)
    for k in [k for k in sys.modules if k == "zippir" or k.startswith("zippir.")]:
        monkeypatch.delitem(sys.modules, k)
    d = str(tmp_path / "hints")
    srv = _server(store_dir=d)
    try:
        from zippir.hintstore import HintStore
        assert isinstance(srv.store, HintStore)
        pk = PaillierPublicKey((1 << 63) + 29, 64)
        cid = srv.register(pk, b"\x07" * 16)
        srv.store.save_hint(cid, 0, 0, [11, 12, 13])
    finally:
        srv.close()
    srv2 = _server(store_dir=d)
    try:
        reg = srv2.registrations[cid]
        assert reg.pk.m == pk.m and reg.seed == b"\x07" * 16
        assert [c.c for c in reg.hints[0].entries] == [11, 12, 13]
    finally:
        srv2.close()


def test_slot_window_trim():
    srv = _server()
    try:
        reg = SimpleNamespace(hints={}, consumed={1})
        for qi in range(5):
            reg.hints[qi] = SimpleNamespace(slots=object(), bases=object())
        srv._trim_slots(reg)      # window = hints_per_client = 2, qi 1 consumed
        kept = sorted(qi for qi, h in reg.hints.items() if h.slots is not None)
        assert kept == [3, 4]
        assert all(h.bases is None for qi, h in reg.hints.items() if qi not in kept)
    finally:
        srv.close()
