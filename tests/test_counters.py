"""The drop-in bumps the counters its caller reads (counters.py:1-63,
test_protocol.py:147-155): with the reference's `zippir.counters` importable,
bumps made by this package show up in zippir.counters.measure()."""

import os
import sys
import types

import pytest

from paper_2603_09190_b200 import counters

REF_SRC = "/root/reference/pkg/src"


def _fresh_ref_counters(monkeypatch):
    for k in [k for k in sys.modules if k == "zippir" or k.startswith("zippir.")]:
        monkeypatch.delitem(sys.modules, k)
    monkeypatch.setattr(counters, "_probed", False)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present")
def test_bumps_reach_reference_counters(monkeypatch):
    monkeypatch.syspath_prepend(REF_SRC)
    _fresh_ref_counters(monkeypatch)
    import zippir.counters as zc
    with zc.measure() as ref_m, counters.measure() as own_m:
        counters.bump("add", 17)
        counters.bump("group_mult", 17)
    assert (ref_m.delta.add, ref_m.delta.group_mult, ref_m.delta.modexp) == (17, 17, 0)
    assert (own_m.delta.add, own_m.delta.group_mult) == (17, 17)


def test_minimal_caller_module(monkeypatch):
    """A caller-side counters module registered as zippir.counters later on
    (the reference package not installed) receives the bumps too."""
    _fresh_ref_counters(monkeypatch)
    seen = []
    mod = types.ModuleType("zippir.counters")
    mod.bump = lambda name, amount=1: seen.append((name, amount))
    monkeypatch.setitem(sys.modules, "zippir.counters", mod)
    counters.bump("add", 3)
    assert seen == [("add", 3)]
    with pytest.raises(AttributeError):
        counters.bump("no_such_counter")
