"""PyTorch-facing wrapper over the SGMV C-ABI (libsgmv_b200.so).

PyTorch is only the plumbing here (device memory, the current stream,
``torch.distributed``); every FLOP runs in the hand-written sm_100a kernels
behind include/lsg_sgmv.h.  Shapes follow the reference (lorasim, sgmv.hpp):

* x ``[s_n, h_in]``, y ``[s_n, h_out]`` -- fp16 / bf16, row-major, any row stride
* ``seg_starts`` int32 ``[n+1]`` = ``Segments::boundaries()`` (sgmv.hpp:28)
* ``seg_slot`` int32 ``[n]``: adapter-pool slot of segment s (replaces ``models[s]``)
* ``AdapterPool``: A ``[slots, layers, h_in, r]``, B ``[slots, layers, r, h_out]``
  (``LoraModel::a`` / ``::b`` layouts, sgmv.hpp:38-48), plus the device
  pointer table the kernels index with (slot, layer).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import KERNEL_BGMV, KERNEL_EXPAND, KERNEL_FUSED, KERNEL_SHRINK, LaunchInfo, WeightTable

_DTYPES = {torch.float16: _lib.LSG_F16, torch.bfloat16: _lib.LSG_BF16}


def _stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _check_i32(t: torch.Tensor, name: str) -> None:
    if t.dtype != torch.int32 or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous int32 CUDA tensor")


class AdapterPool:
    """Device-resident LoRA adapters for one projection site, all layers.

    A slot holds one adapter; ``table`` is the ``lsg_weight_table`` the kernels
    use, with per-slot base pointers in device memory (16-byte aligned).
    """

    def __init__(self, num_slots: int, num_layers: int, h_in: int, h_out: int, rank: int,
                 dtype: torch.dtype = torch.float16, device: str | torch.device = "cuda",
                 a: torch.Tensor | None = None, b: torch.Tensor | None = None):
        if dtype not in _DTYPES:
            raise ValueError("dtype must be torch.float16 or torch.bfloat16")
        self.num_slots, self.num_layers = num_slots, num_layers
        self.h_in, self.h_out, self.rank, self.dtype = h_in, h_out, rank, dtype
        self.a = a if a is not None else torch.zeros(num_slots, num_layers, h_in, rank, dtype=dtype, device=device)
        self.b = b if b is not None else torch.zeros(num_slots, num_layers, rank, h_out, dtype=dtype, device=device)
        assert self.a.shape == (num_slots, num_layers, h_in, rank) and self.a.is_contiguous()
        assert self.b.shape == (num_slots, num_layers, rank, h_out) and self.b.is_contiguous()
        es = self.a.element_size()
        a_base, b_base = self.a.data_ptr(), self.b.data_ptr()
        a_slot, b_slot = num_layers * h_in * rank * es, num_layers * rank * h_out * es
        self.a_ptrs = torch.tensor([a_base + s * a_slot for s in range(num_slots)], dtype=torch.int64,
                                   device=self.a.device)
        self.b_ptrs = torch.tensor([b_base + s * b_slot for s in range(num_slots)], dtype=torch.int64,
                                   device=self.a.device)
        self.table = WeightTable(self.a_ptrs.data_ptr(), self.b_ptrs.data_ptr(), h_in * rank, rank * h_out,
                                 num_slots, num_layers, h_in, h_out, rank, _DTYPES[dtype])

    def load(self, slot: int, a_layers: torch.Tensor, b_layers: torch.Tensor) -> None:
        """Copy one adapter ([layers, h_in, r] and [layers, r, h_out]) into a slot."""
        self.a[slot].copy_(a_layers, non_blocking=True)
        self.b[slot].copy_(b_layers, non_blocking=True)

    def layer_view(self, layer: int) -> "AdapterPool":
        """A one-layer pool whose layer 0 is ``layer`` of this one (same slots, same
        storage; only the device pointer table is new).  Lets sites that live in
        different layers of one pool share a grouped call's layer index."""
        if not 0 <= layer < self.num_layers:
            raise ValueError("layer out of range")
        v = AdapterPool.__new__(AdapterPool)
        v.num_slots, v.num_layers = self.num_slots, 1
        v.h_in, v.h_out, v.rank, v.dtype = self.h_in, self.h_out, self.rank, self.dtype
        v.a, v.b = self.a[:, layer:layer + 1], self.b[:, layer:layer + 1]
        es = self.a.element_size()
        v.a_ptrs = self.a_ptrs + layer * self.h_in * self.rank * es
        v.b_ptrs = self.b_ptrs + layer * self.rank * self.h_out * es
        v.table = WeightTable(v.a_ptrs.data_ptr(), v.b_ptrs.data_ptr(), self.h_in * self.rank, self.rank * self.h_out,
                              self.num_slots, 1, self.h_in, self.h_out, self.rank, _DTYPES[self.dtype])
        return v

    @property
    def slot_bytes_per_layer(self) -> int:
        return (self.h_in * self.rank + self.rank * self.h_out) * self.a.element_size()


def _rows_check(x: torch.Tensor | None, y: torch.Tensor | None, pool: AdapterPool):
    for t, name, cols in ((x, "x", pool.h_in), (y, "y", pool.h_out)):
        if t is None:
            continue
        if t.dtype != pool.dtype or not t.is_cuda or t.dim() != 2 or t.stride(1) != 1 or t.shape[1] != cols:
            raise ValueError(f"{name} must be a CUDA [rows, {cols}] {pool.dtype} tensor with unit column stride")


def call_opts(pdl: bool | None = None, tc_min_rows: int | None = None,
              no_tensor_cores: bool | None = None, mma_min_rows: int | None = None) -> "_lib.CallOpts":
    """Per-call options (``lsg_call_opts``); ``None`` keeps the process default."""
    return _lib.CallOpts(-1 if pdl is None else int(bool(pdl)), -1 if tc_min_rows is None else int(tc_min_rows),
                         -1 if no_tensor_cores is None else int(bool(no_tensor_cores)),
                         -1 if mma_min_rows is None else int(mma_min_rows))


def sgmv(y: torch.Tensor, x: torch.Tensor, pool: AdapterPool, seg_starts: torch.Tensor,
         seg_slot: torch.Tensor, layer: int, num_segments: int | None = None, *, pdl: bool | None = None,
         tc_min_rows: int | None = None, no_tensor_cores: bool | None = None,
         mma_min_rows: int | None = None) -> torch.Tensor:
    """y += x . A_slot . B_slot per segment (fused shrink+expand, one launch).

    ``pdl`` / ``tc_min_rows`` / ``no_tensor_cores`` / ``mma_min_rows`` override the process
    defaults (``set_option``) for this call only (``lsg_sgmv_ex``)."""
    _rows_check(x, y, pool)
    _check_i32(seg_starts, "seg_starts")
    _check_i32(seg_slot, "seg_slot")
    n = seg_slot.numel() if num_segments is None else num_segments
    # Segments of >= 128 rows run on the tensor cores and may keep v in a workspace;
    # it comes from torch's caching allocator (stream-ordered, graph-capture safe).
    wsb = sgmv_workspace_size(pool, x.shape[0])
    ws = torch.empty(wsb, dtype=torch.uint8, device=x.device) if wsb else None
    opts = call_opts(pdl, tc_min_rows, no_tensor_cores, mma_min_rows)
    _lib.call("lsg_sgmv_ex", _ptr(y), y.stride(0), _ptr(x), x.stride(0), C.byref(pool.table), _ptr(seg_starts),
              _ptr(seg_slot), n, x.shape[0], layer, _ptr(ws) if ws is not None else None, wsb, C.byref(opts),
              _stream())
    return y


def sgmv_multi(ys, xs, pools, seg_starts: torch.Tensor, seg_slot: torch.Tensor, layer: int,
               num_segments: int | None = None, *, pdl: bool | None = None, tc_min_rows: int | None = None):
    """Grouped fused call: ``ys[i] += xs[i] . A_i . B_i`` for up to 8 sites sharing one
    segment plan (e.g. q / k / v of a layer), in one launch (lsg_sgmv_multi)."""
    if not (len(ys) == len(xs) == len(pools)) or not 1 <= len(ys) <= 8:
        raise ValueError("sgmv_multi needs 1..8 sites with one y, x and pool each")
    for y, x, pool in zip(ys, xs, pools):
        _rows_check(x, y, pool)
    _check_i32(seg_starts, "seg_starts")
    _check_i32(seg_slot, "seg_slot")
    n = seg_slot.numel() if num_segments is None else num_segments
    sites = (_lib.Site * len(ys))(*[_lib.Site(y.data_ptr(), y.stride(0), x.data_ptr(), x.stride(0),
                                              C.pointer(pool.table)) for y, x, pool in zip(ys, xs, pools)])
    opts = call_opts(pdl, tc_min_rows)
    _lib.call("lsg_sgmv_multi_ex", sites, len(ys), _ptr(seg_starts), _ptr(seg_slot), n, xs[0].shape[0], layer,
              C.byref(opts), _stream())
    return ys


def dense_lora(y: torch.Tensor, x: torch.Tensor, w: torch.Tensor, pool: AdapterPool, seg_starts: torch.Tensor,
               seg_slot: torch.Tensor, layer: int, num_segments: int | None = None) -> torch.Tensor:
    """``y = x . W + x . A_slot . B_slot`` (overwrite): the dense projection with the LoRA add
    in the GEMM epilogue (lsg_dense_lora; rank 16, <= 64 rows).  W is ``[h_in, h_out]``."""
    _rows_check(x, y, pool)
    _check_i32(seg_starts, "seg_starts")
    _check_i32(seg_slot, "seg_slot")
    if w.dtype != pool.dtype or not w.is_cuda or w.dim() != 2 or w.stride(1) != 1 or \
            tuple(w.shape) != (pool.h_in, pool.h_out):
        raise ValueError(f"w must be a CUDA [{pool.h_in}, {pool.h_out}] {pool.dtype} tensor with unit column stride")
    n = seg_slot.numel() if num_segments is None else num_segments
    wsb = int(_lib.lib().lsg_dense_lora_workspace_size(C.byref(pool.table), x.shape[0]))
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=x.device)
    _lib.call("lsg_dense_lora", _ptr(y), y.stride(0), _ptr(x), x.stride(0), _ptr(w), w.stride(0), C.byref(pool.table),
              _ptr(seg_starts), _ptr(seg_slot), n, x.shape[0], layer, _ptr(ws), ws.numel(), _stream())
    return y


def sgmv_workspace_size(pool: AdapterPool, rows: int) -> int:
    """Bytes of workspace a fused call over ``rows`` rows may use (0: none)."""
    return int(_lib.lib().lsg_sgmv_workspace_size(C.byref(pool.table), rows))


def sgmv_shrink(v: torch.Tensor, x: torch.Tensor, pool: AdapterPool, seg_starts: torch.Tensor,
                seg_slot: torch.Tensor, layer: int, num_segments: int | None = None) -> torch.Tensor:
    """v = x . A_slot per segment; v fp32 ``[s_n, r]`` (overwritten)."""
    _rows_check(x, None, pool)
    if v.dtype != torch.float32 or not v.is_contiguous() or tuple(v.shape) != (x.shape[0], pool.rank):
        raise ValueError("v must be a contiguous fp32 [rows, rank] CUDA tensor")
    n = seg_slot.numel() if num_segments is None else num_segments
    _lib.call("lsg_sgmv_shrink", _ptr(v), _ptr(x), x.stride(0), C.byref(pool.table), _ptr(seg_starts),
              _ptr(seg_slot), n, x.shape[0], layer, _stream())
    return v


def sgmv_expand(y: torch.Tensor, v: torch.Tensor, pool: AdapterPool, seg_starts: torch.Tensor,
                seg_slot: torch.Tensor, layer: int, num_segments: int | None = None) -> torch.Tensor:
    """y += v . B_slot per segment."""
    _rows_check(None, y, pool)
    if v.dtype != torch.float32 or not v.is_contiguous() or tuple(v.shape) != (y.shape[0], pool.rank):
        raise ValueError("v must be a contiguous fp32 [rows, rank] CUDA tensor")
    n = seg_slot.numel() if num_segments is None else num_segments
    _lib.call("lsg_sgmv_expand", _ptr(y), y.stride(0), _ptr(v), C.byref(pool.table), _ptr(seg_starts),
              _ptr(seg_slot), n, y.shape[0], layer, _stream())
    return y


def bgmv(y: torch.Tensor, x: torch.Tensor, pool: AdapterPool, row_slot: torch.Tensor, layer: int) -> torch.Tensor:
    """Decode BGMV: y[i] += x[i] . A_{row_slot[i]} . B_{row_slot[i]} (negative slot = no adapter)."""
    _rows_check(x, y, pool)
    _check_i32(row_slot, "row_slot")
    _lib.call("lsg_bgmv", _ptr(y), y.stride(0), _ptr(x), x.stride(0), C.byref(pool.table), _ptr(row_slot),
              x.shape[0], layer, _stream())
    return y


def build_segments(row_slot: torch.Tensor, num_slots: int, lead_slot: int = -1, lead_rows: tuple[int, int] = (0, 0)):
    """On-device stable grouping of rows by slot (plan_batch's order, simulator.cpp:239-311).

    ``lead_slot``: the prefill request's slot (its group goes first); ``lead_rows``: that
    request's own row range [r0, r1) in ``row_slot`` (placed ahead of the same-adapter
    decode rows).  Returns (row_perm [s_n], seg_starts [s_n+1], seg_slot [s_n],
    num_segments [1]) -- all device int32; seg_starts / seg_slot are padded past the
    true segment count.
    """
    _check_i32(row_slot, "row_slot")
    s_n = row_slot.numel()
    dev = row_slot.device
    row_perm = torch.empty(max(s_n, 1), dtype=torch.int32, device=dev)
    seg_starts = torch.empty(s_n + 1, dtype=torch.int32, device=dev)
    seg_slot = torch.empty(max(s_n, 1), dtype=torch.int32, device=dev)
    nseg = torch.empty(1, dtype=torch.int32, device=dev)
    _lib.call("lsg_build_segments", _ptr(row_slot), s_n, num_slots, lead_slot, int(lead_rows[0]), int(lead_rows[1]),
              _ptr(row_perm), _ptr(seg_starts),
              _ptr(seg_slot), _ptr(nseg), None, 0, _stream())
    return row_perm[:s_n], seg_starts, seg_slot[:s_n], nseg


def gather_rows(dst: torch.Tensor, src: torch.Tensor, row_perm: torch.Tensor) -> torch.Tensor:
    """dst[i] = src[row_perm[i]] for 16-bit rows."""
    _lib.call("lsg_gather_rows", _ptr(dst), dst.stride(0), _ptr(src), src.stride(0), _ptr(row_perm),
              row_perm.numel(), dst.shape[1], _stream())
    return dst


def scatter_rows(dst: torch.Tensor, src: torch.Tensor, row_perm: torch.Tensor) -> torch.Tensor:
    """dst[row_perm[i]] = src[i] for 16-bit rows."""
    _lib.call("lsg_scatter_rows", _ptr(dst), dst.stride(0), _ptr(src), src.stride(0), _ptr(row_perm),
              row_perm.numel(), dst.shape[1], _stream())
    return dst


def set_option(option: int, value: int) -> None:
    _lib.call("lsg_set_option", option, value)


def get_option(option: int) -> int:
    return _lib.lib().lsg_get_option(option)


def query_launch(pool: AdapterPool, num_segments: int, total_rows: int, kernel: int = KERNEL_FUSED) -> dict:
    info = LaunchInfo()
    _lib.call("lsg_query_launch", C.byref(pool.table), num_segments, total_rows, kernel, C.byref(info))
    return {f: getattr(info, f) for f, _ in LaunchInfo._fields_}


__all__ = ["AdapterPool", "call_opts", "sgmv", "sgmv_multi", "dense_lora", "sgmv_shrink", "sgmv_expand", "bgmv", "build_segments", "gather_rows",
           "scatter_rows", "set_option", "get_option", "query_launch", "KERNEL_FUSED", "KERNEL_SHRINK",
           "KERNEL_EXPAND", "KERNEL_BGMV"]
