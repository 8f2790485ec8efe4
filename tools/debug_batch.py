import os, sys, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import Golden
import paper_2603_09190_b200 as z
from paper_2603_09190_b200 import device
from paper_2603_09190_b200.bigint import key_ctx, ints_to_limbs
from oracle import client
g = Golden("tiny")
st = z.ServerGlobalState(g.params(z), g.db)
dev = st.device; lay = st.layout
rng = random.Random(5)
nq = 5
keys = [client.SecretKey(g.p, g.q)] + [client.keygen(2048, random.Random(1000 + j)) for j in range(2)]
qus = [np.array([rng.randrange(1 << 32) for _ in range(g.d0)], dtype=np.uint64) for _ in range(nq)]
cks = [[rng.randrange(keys[i % 3].m) for _ in range(1024)] for i in range(nq)]
ks = [key_ctx(keys[i % 3].m, dev) for i in range(nq)]
q32 = np.zeros((nq, lay.ld), np.uint32)
for i in range(nq): q32[i, :g.d0] = qus[i]
qd = device.u32_tensor(q32, dev).reshape(nq, lay.ld)
planes = device.query_planes(qd, 256)
b = device.to_host_u32(device.umma_gemv(st.dbt, planes, nq))
for i in range(nq):
    bi = st.db_matvec(qus[i])
    print("b", i, np.array_equal(b[i, :g.d1].astype(np.uint64), bi))
cko = np.stack([ints_to_limbs(cks[i], 64) for i in range(nq)])
cd = device.u32_tensor(cko, dev).reshape(nq, 1024, 64)
bc = device.build_bc_batch(cd, 64)
for i in range(nq):
    bci = device.build_bc(cd[i].contiguous(), 64)
    print("bc", i, torch.equal(bc[i], bci))
zb = device.umma_answer_rows_batch(st.H_dev, bc, 64)
for i in range(nq):
    bci = device.build_bc(cd[i].contiguous(), 64)
    zi = device.umma_answer_rows(st.H_dev, bci, torch.zeros(lay.rows, dtype=torch.int32, device=dev), 0xFFFFFFFF, 64)
    print("z", i, torch.equal(zb[i], zi))
bd = device.u32_tensor(b, dev).reshape(nq, -1)
t = device.to_host_u32(device.answer_groups_batch(zb, bd, 0xFFFFFFFF, lay.d1, lay.cap, lay.groups, ks, 128))
for i in range(nq):
    ti = device.to_host_u32(device.answer_groups(zb[i].contiguous(), bd[i].contiguous(), 0xFFFFFFFF, lay.d1, lay.cap, lay.groups, ks[i], 128))
    print("t", i, np.array_equal(t[i], ti))
