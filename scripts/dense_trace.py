"""Needs the traced build: scripts/build_variant.sh dn_trace -DLSG_DN_TRACE (copied over the
product library). Phase timeline of one lsg_dense_lora launch (the last of a 32-layer CUDA-graph
step): per phase the median / max over CTAs of %globaltimer since the earliest CTA entry."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_18547_b200 as lsg  # noqa: E402

PH = ["entry", "-", "first B rows loaded", "v ready (PDL wait)", "lora blocks filled", "W MMAs issued", "last MMA issued",
      "exit"]


def main():
    h, r, rows, L = 4096, 16, 64, 32
    lsg.set_option(lsg.LSG_OPT_PDL, 1)
    dt = torch.float16
    pool = lsg.AdapterPool(rows, L, h, h, r, dt)
    pool.a.uniform_(-1, 1)
    pool.b.uniform_(-1, 1)
    Ws = torch.empty(L, h, h, dtype=dt, device="cuda").uniform_(-0.05, 0.05)
    xs = torch.empty(L, rows, h, dtype=dt, device="cuda").uniform_(-1, 1)
    ys = torch.zeros(L, rows, h, dtype=dt, device="cuda")
    ss = torch.arange(rows + 1, dtype=torch.int32, device="cuda")
    sl = torch.arange(rows, dtype=torch.int32, device="cuda")
    st = torch.cuda.Stream()

    import ctypes as C
    from paper_2310_18547_b200 import _lib
    wsb = int(_lib.lib().lsg_dense_lora_workspace_size(C.byref(pool.table), rows))
    ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")

    def fused():
        for l in range(L):
            _lib.call("lsg_dense_lora", ys[l].data_ptr(), h, xs[l].data_ptr(), h, Ws[l].data_ptr(), h,
                      C.byref(pool.table), ss.data_ptr(), sl.data_ptr(), rows, rows, l, ws.data_ptr(), wsb,
                      C.c_void_p(torch.cuda.current_stream().cuda_stream))
    with torch.cuda.stream(st):
        fused()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fused()
        for _ in range(5):
            g.replay()
    torch.cuda.synchronize()
    off = 64 * 16 * 4
    allt = ws[off:off + 2 * 220 * 8 * 8].cpu().numpy().view(np.uint64).reshape(2, 220, 8).astype(np.int64)
    # layer 31 (slot 1) against layer 30 (slot 0): the step between two launches
    d0, d1 = allt[0][:128], allt[1][:128]
    s1 = allt[1][148:148 + rows]
    t0 = d1[:, 0].min()
    print(f"previous GEMM exit (max over CTAs)  {(d0[:, 7].max() - t0) / 1e3:8.2f} us")
    for i, name in enumerate(["shrink entry", "shrink wait done", "shrink FMAs done", "shrink exit"]):
        v = s1[:, i] - t0
        print(f"{name:26s} median {np.median(v) / 1e3:7.2f} us  max {v.max() / 1e3:7.2f} us  min {v.min() / 1e3:7.2f}")
    for i, name in enumerate(PH):
        v = d1[:, i]
        v = v[v > 0] - t0
        if len(v):
            print(f"{name:26s} median {np.median(v) / 1e3:7.2f} us  max {v.max() / 1e3:7.2f} us  min {v.min() / 1e3:7.2f}")


if __name__ == "__main__":
    main()
