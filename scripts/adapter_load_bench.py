"""On-demand adapter loading on the B200 against the
reference's model of it (cost_model.cpp:91-100: 7 projections x (A+B) per layer
over PCIe, anchors ~50 us/layer and ~2 ms/model, test_cost_model.cpp:134-145).

Prints one JSON line: H2D time per layer and per adapter (pinned host -> pool
slot, copy stream), and the SGMV decode step time alone vs. with adapter loads
running concurrently on the copy stream.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_18547_b200 as lsg  # noqa: E402
from paper_2310_18547_b200.adapters import AdapterStore  # noqa: E402


def main():
    h, r, layers, sites = 4096, 16, 32, 7
    store = AdapterStore([(h, h)] * sites, num_slots=4, num_layers=layers, rank=r, dtype=torch.float16)
    compute_pools = [lsg.AdapterPool(64, layers, h, h, r, torch.float16) for _ in range(sites)]  # the step's adapters
    host = [(torch.randn(layers, h, r, dtype=torch.float16).pin_memory(),
             torch.randn(layers, r, h, dtype=torch.float16).pin_memory()) for _ in range(sites)]
    per_adapter = store.bytes_per_adapter
    # warm-up load
    store.load(-1, host)
    torch.cuda.synchronize()
    n = 8
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(store.copy_stream)
    for i in range(n):
        store.load(i, host)
    e1.record(store.copy_stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    # SGMV step (64 distinct rows, every site of every layer) alone and under loads
    lsg.set_option(lsg.LSG_OPT_PDL, 1)
    x = torch.randn(64, h, dtype=torch.float16, device="cuda")
    y = torch.zeros(64, h, dtype=torch.float16, device="cuda")
    ss = torch.arange(65, dtype=torch.int32, device="cuda")
    sl = torch.arange(64, dtype=torch.int32, device="cuda")
    comp = torch.cuda.Stream()

    def step():
        for layer in range(layers):
            for p in compute_pools:
                lsg.sgmv(y, x, p, ss, sl, layer)

    with torch.cuda.stream(comp):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=comp):
        step()

    def timed(k, loads):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(comp):
            a.record(comp)
            for i in range(k):
                if loads:
                    store.load(1000 + i, host)
                g.replay()
            b.record(comp)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / k

    timed(3, False)
    alone = timed(20, False)
    with_loads = timed(20, True)
    print(json.dumps({
        "adapter_bytes": per_adapter, "bytes_per_layer": per_adapter // layers,
        "h2d_ms_per_adapter": ms, "h2d_us_per_layer": ms * 1e3 / layers,
        "h2d_gbs": per_adapter / (ms * 1e-3) / 1e9,
        "reference_model_us_per_layer": "adapter_load_latency(1) ~ 50 (PCIe Gen4 model, test_cost_model.cpp:134-145)",
        "sgmv_step_ms_alone": alone, "sgmv_step_ms_with_concurrent_loads": with_loads,
        "step": f"{layers * sites} fused SGMV launches (h={h}, r={r}, 64 distinct rows), CUDA graph, PDL"}))


if __name__ == "__main__":
    main()
