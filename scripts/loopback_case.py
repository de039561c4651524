"""One loopback slab-decomposition case against the oracle, in its own process (a
kernel fault cannot take other cases with it): prints OK / FAIL.
Usage: python scripts/loopback_case.py PEER_HALO NRANKS NX NY M ROWS [SOR_FUSE]
(PEER_HALO 0/1 -> IBM_PEER_HALO; ROWS -> IBM_WF_ROWS, 0 = the library's choice).
Set IBM_DEBUG_SYNC=1 to locate a faulting kernel (a sync and check after each phase)."""
import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import ibm_inputs as I
from test_gpu_parity import assert_parity, run_pair
from oracle import oracle as O
import paper_2402_17337_b200 as P
peer, Pn, nx, ny, m, rows = sys.argv[1:7]
fuse = int(sys.argv[7]) if len(sys.argv) > 7 else int(m)
os.environ["IBM_PEER_HALO"] = peer
if int(rows): os.environ["IBM_WF_ROWS"] = rows
cfg = I.cfg1(nx=int(nx), ny=int(ny), steps=3, maxit_p=700)
try:
    o, g, ro, rg = run_pair((O, P), cfg, cfg.steps, nranks=int(Pn), loopback=True, sor_batch=5, sor_fuse=fuse)
    assert_parity(o, g, ro, rg)
    try:
        ph = g.query("peer_halo")
    except Exception:
        ph = "-"
    print("OK", sys.argv[1:], ph, os.environ.get("IBM_LIB_VARIANT", ""))
except Exception as e:
    print("FAIL", sys.argv[1:], os.environ.get("IBM_LIB_VARIANT", ""), repr(e)[:300])
