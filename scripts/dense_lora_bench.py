""" Dense projection + LoRA: the fused kernel (lsg_dense_lora: tcgen05 GEMM
with the LoRA add in its epilogue, after the shrink) against the unfused baseline
(cuBLAS GEMM x.W, then the fused SGMV kernel accumulating the LoRA into its output).
Llama-2-7B projection shape, 64 decode rows, Distinct adapters; 32 (W, adapter-layer) pairs
rotated per step so W (32 MiB each) and the adapters stream from HBM; CUDA graph, PDL.
Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_18547_b200 as lsg  # noqa: E402


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

    def fused():
        for l in range(L):
            lsg.dense_lora(ys[l], xs[l], Ws[l], pool, ss, sl, l)

    def unfused():
        for l in range(L):
            torch.mm(xs[l], Ws[l], out=ys[l])
            lsg.sgmv(ys[l], xs[l], pool, ss, sl, l)

    def gemm_only():
        for l in range(L):
            torch.mm(xs[l], Ws[l], out=ys[l])

    def gemm_kmajor():  # the same GEMM on W stored [h_out, h_in] (nn.Linear layout), for reference
        for l in range(L):
            torch.mm(xs[l], Ws[l].t(), out=ys[l])

    if "--profile" in sys.argv:  # ncu: a few plain launches of each variant, no graph
        for fn in (fused, unfused, gemm_only):
            fn()
        torch.cuda.synchronize()
        return
    out = {}
    for name, fn in (("fused_us", fused), ("unfused_us", unfused), ("cublas_gemm_only_us", gemm_only),
                     ("cublas_gemm_w_kmajor_us", gemm_kmajor)):
        with torch.cuda.stream(st):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
        with torch.cuda.stream(st):
            for _ in range(3):
                g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(20):
                g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) * 1e3 / (20 * L)
    bytes_ = h * h * 2 + 2 * rows * h * 2 + 2 * (rows * (h + r) + rows * h * r) * 2  # W + x,y + LoRA pair
    out.update({"shape": f"x[{rows},{h}] . W[{h},{h}] + LoRA r={r}, {rows} distinct adapters, fp16",
                "alg_bytes": bytes_, "fused_gbs": bytes_ / out["fused_us"] / 1e3})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
