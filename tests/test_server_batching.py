"""Host logic of the batched hint worker (server.py:_generate_hints) on CPU:
a batch of queued (client, qi) jobs becomes ONE protocol.hints call for the
jobs without a usable slot decomposition and ONE protocol.refresh_hints call
per distinct changed-row set for the stale ones; fresh hints and unknown
clients are skipped; results land in the registrations. protocol's device
functions are replaced by recorders (no GPU needed)."""

from types import SimpleNamespace

import numpy as np

from paper_2603_09190_b200 import protocol, server


def _hint(qi, version, slots=None):
    return SimpleNamespace(query_index=qi, db_version=version, slots=slots, entries=[],
                           dev=None, bases=None)


def test_generate_hints_groups_jobs(monkeypatch):
    params = SimpleNamespace(hints_per_client=3)
    state = SimpleNamespace(db_version=2, device="cpu")
    srv = server.PirServer(params, None, state=state, hint_workers=1)
    try:
        regs = {}
        for c in (b"a", b"b", b"c"):
            regs[c] = SimpleNamespace(client_id=c, hints={}, consumed=set())
        # a: stale hint with slots at version 1 (delta 1->2 known), b: stale at
        # version 0 (deltas 1 and 2 known), c: fresh hint for qi 0, none for qi 1
        regs[b"a"].hints[0] = _hint(0, 1, slots=object())
        regs[b"b"].hints[0] = _hint(0, 0, slots=object())
        regs[b"c"].hints[0] = _hint(0, 2)
        srv.registrations.update(regs)
        srv._deltas = {1: np.array([5, 9]), 2: np.array([9, 40])}
        calls = {"hints": [], "refresh": []}

        def fake_hints(st, jobs, stream=None, keep_slots=False):
            calls["hints"].append([(r.client_id, qi) for r, qi in jobs])
            return [_hint(qi, st.db_version) for _, qi in jobs]

        def fake_refresh(st, pairs, rows, stream=None):
            calls["refresh"].append(([r.client_id for r, _ in pairs], list(rows)))
            return [_hint(old.query_index, st.db_version) for _, old in pairs]

        monkeypatch.setattr(protocol, "hints", fake_hints)
        monkeypatch.setattr(protocol, "refresh_hints", fake_refresh)
        srv._generate_hints([(b"a", 0), (b"b", 0), (b"c", 0), (b"c", 1), (b"c", 1),
                             (b"zz", 0)])
        assert calls["hints"] == [[(b"c", 1)]]
        assert sorted(calls["refresh"]) == [([b"a"], [9, 40]), ([b"b"], [5, 9, 40])]
        assert all(h.db_version == 2 for r in regs.values() for h in r.hints.values())
        assert set(regs[b"c"].hints) == {0, 1}
    finally:
        srv.close()
