"""Timeline of the host-buffer apply pipeline (Operator.apply_host on a
pinned CPU tensor, config 5): CUDA-event timestamps of every H2D chunk,
volume group and D2H chunk relative to the first H2D, to see where the
end-to-end time goes against the PCIe ceiling (tools/pcie_probe.py)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal  # noqa: E402
from paper_1709_06793_b200 import _lib  # noqa: E402
from paper_1709_06793_b200._lib import check, lib  # noqa: E402
from paper_1709_06793_b200.shard import slab_mesh  # noqa: E402
from tests.cases import k_c5  # noqa: E402

g = RefinedGrid(slab_mesh(0, 1), 8)
op = Operator(g, "scaling", sample_nodal(k_c5(), g), fast=True)
u = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, g.n_nodes)).pin_memory()
for _ in range(3):
    r = op.apply(u)
    del r
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    r = op.apply(u)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
    del r
print("apply_host ms", [round(x, 2) for x in ts], flush=True)

# instrumented copy of apply_host
D = op._device()
P = op._pipeline()
dg, ds = D["grid"], D["surf"]
h2d, comp, d2h = P["streams"]
du, out = P["du"], P["out"]
chunks = op._chunks()
flags = op._vol_flags(residual=False)


def ev(s):
    e = torch.cuda.Event(enable_timing=True)
    e.record(s)
    return e


d2h_b = torch.cuda.Stream()


def run(lag, verbose=False, nd2h=1):
    hout = torch.empty(g.n_nodes, dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()
    t_host0 = time.perf_counter()
    cur = torch.cuda.current_stream()
    for st in P["streams"]:
        st.wait_stream(cur)
    e0 = ev(h2d)
    ev_in = [None] * len(chunks)
    ev_out = []

    def put(ci):
        a, b = chunks[ci]
        with torch.cuda.stream(h2d):
            if lag and ci - 2 - lag >= 0:
                h2d.wait_event(ev_out[ci - 2 - lag])
            if b > a:
                du[a:b].copy_(u[a:b], non_blocking=True)
            ev_in[ci] = ev(h2d)
    nput = min(len(chunks), 2 + lag) if lag else len(chunks)
    for ci in range(nput):
        put(ci)
    comp.wait_event(ev_in[0])
    cs = comp.cuda_stream
    check(lib.hhg_ghost_update(dg.ref, du.data_ptr(), cs))
    t_comp = []
    for gi, desc in enumerate(P["descs"]):
        comp.wait_event(ev_in[gi + 1])
        check(lib.hhg_volume_apply(P["byref"](desc), op._vol_variant(), flags,
                                   D["coef"].data_ptr(), None, du.data_ptr(), None,
                                   out.data_ptr(), cs))
        e = ev(comp)
        t_comp.append(e)
        sd = d2h if (nd2h == 1 or gi % 2 == 0) else d2h_b
        sd.wait_event(e)
        a, b = chunks[gi + 1]
        with torch.cuda.stream(sd):
            hout[a:b].copy_(out[a:b], non_blocking=True)
        ev_out.append(ev(sd))
        if lag and nput < len(chunks):
            put(nput)
            nput += 1
    op._surface(dg, ds, 0, du, None, out, cs)
    e = ev(comp)
    d2h.wait_event(e)
    a, b = chunks[0]
    with torch.cuda.stream(d2h):
        hout[a:b].copy_(out[a:b], non_blocking=True)
    d2h.wait_stream(d2h_b)
    e_end = ev(d2h)
    d2h.synchronize()
    t_host = (time.perf_counter() - t_host0) * 1e3
    rel = lambda e: round(e0.elapsed_time(e), 2)   # noqa: E731
    ok = torch.equal(hout, ref)
    print(f"lag {lag} d2h streams {nd2h}: host {t_host:.2f} ms, device end {rel(e_end)} ms, equal {ok}", flush=True)
    if verbose:
        print("  h2d chunk ends", [rel(e) for e in ev_in[::4]], "last", rel(ev_in[-1]))
        print("  comp ends     ", [rel(e) for e in t_comp[::4]], "last", rel(t_comp[-1]))
        print("  d2h ends      ", [rel(e) for e in ev_out[::4]], "last", rel(ev_out[-1]))
    del hout


ref = op.apply(u).clone()
for lag, nd in ((0, 1), (0, 2), (1, 2), (2, 2)):
    for rep in range(3):
        run(lag, verbose=rep == 2, nd2h=nd)
