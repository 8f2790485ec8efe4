"""PirServer mirror on the GPU: background hint worker, look-ahead window,
database update with stale-hint regeneration (reference server.py:62-124;
tests test_protocol.py:56-71 update replay, test_acceptance.py:333-360
silent offline)."""

import random

import numpy as np
import pytest

from oracle import client

pytestmark = pytest.mark.gpu


def test_server_update_and_regenerate():
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200.server import HintPending, PirServer
    rng = random.Random(31)
    params = z.ProtocolParams(z.LweParams(n=64, q=1 << 32, p=256, noise_sigma=6.4), 32, 48, 768,
                              hints_per_client=3)
    db = np.array([[rng.randrange(256) for _ in range(48)] for _ in range(32)])
    srv = PirServer(params, db)
    try:
        sk, seed = client.setup(768, rng)
        pk = z.PaillierPublicKey(sk.m, sk.m.bit_length())
        cid = srv.register(pk, seed)
        srv.wait_for_hints(timeout=120)
        reg = srv.registrations[cid]
        assert sorted(reg.hints) == [0, 1, 2]
        A = srv.state.A

        def ask(qi, i0, mode):
            qu0, ck_o, _ = client.query(sk, seed, 64, 1 << 32, 256, 6.4, 32, i0, qi, rng, A)
            r = srv.answer(cid, z.QueryMessage(cid, qi, mode, ck_o, qu0))
            if mode == z.SEPARATE:
                return client.extract(sk, 1 << 32, 256, params.capacity, 1 << 32, 48,
                                      t=r.t, k=[c.c for c in r.k])
            return client.extract(sk, 1 << 32, 256, params.capacity, 1 << 32, 48,
                                  combined=[c.c for c in r.k])

        assert ask(0, 5, z.SEPARATE) == [int(x) for x in db[5]]
        # database update: hints go stale, the worker regenerates them silently
        db2 = np.array([[rng.randrange(256) for _ in range(48)] for _ in range(32)])
        srv.update_database(db2)
        assert srv.state.db_version == 1
        srv.wait_for_hints(timeout=120)
        assert all(h.db_version == 1 for h in reg.hints.values())
        assert ask(1, 7, z.COMBINED) == [int(x) for x in db2[7]]
        # a query index outside the window is pending, then served
        with pytest.raises(HintPending):
            ask(9, 0, z.SEPARATE)
        srv.wait_for_hints(timeout=120)
        assert ask(9, 3, z.SEPARATE) == [int(x) for x in db2[3]]
    finally:
        srv.close()
