"""Debug: lsg_dense_lora vs cuBLAS + lsg_sgmv on one problem; per-row error and the shrink's v."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_18547_b200 as lsg  # noqa: E402
from paper_2310_18547_b200 import _lib  # noqa: E402
from tests._util import UNIFORM, DISTINCT, segments_for  # noqa: E402


def run(pop, batch, h_in, h_out):
    torch.manual_seed(0)
    r = 16
    bounds, _, _ = segments_for(pop, batch, 44)
    n = len(bounds) - 1
    pool = lsg.AdapterPool(n, 1, h_in, h_out, r, torch.float16)
    pool.a.uniform_(-1, 1)
    pool.b.uniform_(-1, 1)
    x = torch.empty(batch, h_in, dtype=torch.float16, device="cuda").uniform_(-1, 1)
    W = torch.empty(h_in, h_out, dtype=torch.float16, device="cuda").uniform_(-0.05, 0.05)
    ss = torch.tensor(bounds.astype("int64"), dtype=torch.int32, device="cuda")
    sl = torch.arange(n, dtype=torch.int32, device="cuda")
    wsb = int(_lib.lib().lsg_dense_lora_workspace_size(C.byref(pool.table), batch))
    ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
    y = torch.full((batch, h_out), float("nan"), dtype=torch.float16, device="cuda")
    _lib.call("lsg_dense_lora", y.data_ptr(), h_out, x.data_ptr(), h_in, W.data_ptr(), h_out, C.byref(pool.table),
              ss.data_ptr(), sl.data_ptr(), n, batch, 0, ws.data_ptr(), wsb, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    v = ws.view(torch.float32)[:batch * r].view(batch, r)
    v2 = torch.empty(batch, r, dtype=torch.float32, device="cuda")
    lsg.sgmv_shrink(v2, x, pool, ss, sl, 0)
    y2 = (x.float() @ W.float()).half()
    lsg.sgmv(y2, x, pool, ss, sl, 0)
    torch.cuda.synchronize()
    ev = ((v - v2).abs().max(1).values / v2.abs().max(1).values.clamp_min(1e-9)).cpu()
    ey = ((y.float() - y2.float()).abs().max(1).values / y2.float().abs().max(1).values).cpu()
    print(pop, batch, h_in, h_out, "segments", n, "bounds", bounds.tolist()[:12])
    print(" v rel err per row:", [round(float(e), 4) for e in ev])
    print(" y rel err per row:", [round(float(e), 4) for e in ey])
    bad = (y.float() - y2.float()).abs() > 0.05 * y2.float().abs().max()
    if bad.any():
        cols = bad.any(0).nonzero().flatten().cpu().tolist()
        print(" bad columns:", cols[:20], "... count", len(cols))
        import collections
        print(" by tile:", sorted(collections.Counter(c // 128 for c in cols).items()))
        print(" by owner slice (16 cols):", sorted(collections.Counter((c % 128) // 16 for c in cols).items()))
        rows = bad.any(1).nonzero().flatten().cpu().tolist()
        print(" bad rows:", rows)


if __name__ == "__main__":
    lsg.set_option(lsg.LSG_OPT_PDL, int(os.environ.get("PDL", "0")))
    run(UNIFORM, 37, 4096, 2048)
    run(DISTINCT, 64, 4096, 4096)
