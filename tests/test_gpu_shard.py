"""The row-sharded server on real device kernels: two ranks (processes) each
build their group-aligned shard (ShardedServer: DB slice, H slice, local
groups incl. the partial last group) and answer a query with respond(); the
per-shard t rows, assembled by shard.gather_groups over gloo, equal the
single-process answer of the whole DB. Both processes share the one GPU of
this box; their kernels are independent (no cross-process waiting), only the
host-side gather is collective."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

D0, D1, N = 2048, 4000, 1024


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    import random
    from oracle import client
    rng = np.random.default_rng(77)
    db = rng.integers(0, 256, (D0, D1), dtype=np.uint8)
    qu = rng.integers(0, 1 << 32, D0, dtype=np.uint64)
    sk = client.keygen(2048, random.Random(78))
    r = random.Random(79)
    ck = [r.randrange(sk.m) for _ in range(N)]
    return db, qu, sk.m, ck


def _t_of(z, st, m, ck, qu, groups):
    pk = z.PaillierPublicKey(m, m.bit_length())
    reg = z.ClientRegistration(pk, b"\x01" * 16, z.client_id_of(pk))
    reg.hints[0] = z.ClientHint(0, st.db_version, [z.PaillierCiphertext(1)] * groups)
    return z.respond(st, reg, z.QueryMessage(reg.client_id, 0, z.SEPARATE, ck, qu)).t


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200.bigint import ints_to_limbs, limbs_to_ints
    from paper_2603_09190_b200.shard import ShardedServer, gather_groups, shard_bounds
    db, qu, m, ck = _inputs()
    params = z.ProtocolParams(z.LweParams(N, 1 << 32, 256, 6.4), D0, D1, 2048)
    bounds = shard_bounds(D1, params.capacity, world)
    lo, hi, glo, ghi = bounds[rank]
    srv = ShardedServer(params, np.ascontiguousarray(db[:, lo:hi]), rank, world)
    t = _t_of(z, srv.state, m, ck, qu, ghi - glo)
    L = 64
    local = torch.from_numpy(ints_to_limbs(t, L).view(np.int32))
    full = gather_groups(local, bounds, rank)
    got = limbs_to_ints(full.numpy().view(np.uint32))
    if rank == 0:
        st = z.ServerGlobalState(params, db)
        out.put(got == _t_of(z, st, m, ck, qu, params.d1_prime))
    dist.destroy_process_group()


def test_two_shards_on_device_match_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert ok
    assert all(p.exitcode == 0 for p in procs)


def test_sharded_pirserver_full_api_on_device():
    """ShardedPirServer with the real rank-local device path (DeviceShard: the
    shard's ServerGlobalState, tensor-core / IMAD hints, respond on the
    device) on two ranks sharing this box's GPU, gloo command channels:
    register -> hint worker -> answer() and handle_frame() in both modes ->
    update_database (1% of the rows, incremental per shard) -> regenerated
    hints -> answers, all bit-exact against the single-process oracle and
    decoding to the requested record (tests/test_shard_server_gloo.py's
    driver with DeviceShard instead of the CPU oracle)."""
    from test_shard_server_gloo import run_two_ranks
    run_two_ranks(dict(d0=512, d1=700, n=64, bits=1024, sigma=1.0, local="device",
                       rows=[0, 5, 63, 64, 699, 350, 351]), timeout=600)
