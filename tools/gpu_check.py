"""Quick GPU shakedown: parity of both kernels vs the oracle on small meshes + C2 timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1612_09335_b200 as P
from oracle.mesh import OracleMesh
from oracle import reconstruct as R

def check(d, n, M, jit, V, nsel=None, seed=0):
    nodes, cells, period = gen.box_mesh(d, n, True, jit, 4)
    rng = np.random.default_rng(seed)
    Qin = rng.standard_normal((cells.shape[0], V)) + 3
    ctx = P.setup_context(nodes, cells, period, M, V, device=0)
    perm = ctx.permutation()
    Q = Qin[perm]
    Qd = torch.tensor(Q, device="cuda")
    m = OracleMesh(nodes, cells, period, M)
    sel = range(m.N) if nsel is None else rng.choice(m.N, nsel, replace=False)
    ref = np.array([R.reconstruct_cell(m, int(i), Q, M)["w"] for i in sel])
    out = {}
    for k in ("simple", "pipelined"):
        ctx.set_kernel(k)
        o = ctx.reconstruct(Qd)
        torch.cuda.synchronize()
        out[k] = o.cpu().numpy()[list(sel)]
        err = np.abs(out[k] - ref).max() / np.abs(Q).max()
        print(f"d={d} n={n} M={M} V={V} kernel={k}: max err {err:.3e}", flush=True)
    print("  simple vs pipelined bitwise equal:", np.array_equal(out["simple"], out["pipelined"]))
    dbg = ctx.reconstruct_debug(Qd, np.array(list(sel)[:5]))
    print("  debug w == simple:", np.array_equal(dbg["w"], out["simple"][:5]))

check(2, 16, 2, 0.0, 4)
check(2, 24, 3, 0.2, 4)
check(3, 6, 3, 0.1, 9, nsel=200)
check(3, 6, 2, 0.0, 5, nsel=200)

# C2 timing
w = gen.make("C2")
t = time.time()
ctx = P.setup_context(w["nodes"], w["cells"], w["period"], w["M"], w["V"], device=0)
print("C2 setup s", time.time() - t, ctx.info())
Q = torch.tensor(w["avgs"][ctx.permutation()], device="cuda")
out = torch.empty((ctx.info()["n_owned"], w["V"], ctx.nm), dtype=torch.float64, device="cuda")
for k in ("simple", "pipelined"):
    ctx.set_kernel(k)
    for _ in range(5): ctx.reconstruct(Q, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): ctx.reconstruct(Q, out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    B = ctx.info()["algorithmic_bytes_per_cell"] * ctx.info()["n_owned"]
    print(f"C2 {k}: {ms:.4f} ms  {ctx.info()['n_owned']/ms*1e3:.3e} cells/s  {B/ms/1e6:.1f} GB/s")
