"""Device-resident compressed network loaded from a ``.dthn`` image.

``DeviceModel`` is what ``CompressedModel.to_device`` returns (reference CompressedModel,
model_io.py:46-63, whose layers the reference runs one ``layer_forward`` at a time,
kernel.py:296-320). Loading is B200-first:

* the serialized image goes to HBM in ONE pinned host→device copy (``h2d_bytes``);
* every payload is decoded on the GPU by ``dt_unpack_values`` straight out of the device image
  (unaligned little-endian float32/float64 → aligned fp32 masters, plus the bf16 operand copies
  the tensor-core path reads), then the image is released — no host-side conversion;
* the forward chains the layers on one stream with bf16 intermediates on the tensor-core path
  (fp32 on the FFMA path), each layer with its own workspace so consecutive layers pipeline
  (``forward_pipeline``: layer i+1's W regeneration overlaps layer i's GEMM; the regeneration
  reads only the layer's own factors, never the activations in flight).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .core import as_device_matrix, device, stream_handle
from .errors import ArgumentError, DimensionError
from .factor import FactorPair
from .kernel import _act_code, forward_into, forward_pipeline


class DeviceModel:
    """A multi-layer DeepThin network whose factors live in HBM.

    activations: one name for every layer, or one per layer (default "identity"); act_args:
    the clipped-ReLU ceiling per layer (default 20.0, as layer_forward). mma: "bf16" (tcgen05
    tensor cores, bf16 intermediates) or "ffma" (fp32 CUDA cores, fp32 intermediates).
    """

    def __init__(self, model, activations=None, *, mma: str = "bf16", act_args=None,
                 pipeline: bool = True):
        if mma not in ("bf16", "ffma"):
            raise ArgumentError(f"mma must be 'bf16' or 'ffma', got {mma!r}")
        image, index = model.image()
        count = len(index)
        if activations is None or isinstance(activations, str):
            activations = [activations or "identity"] * count
        if act_args is None or isinstance(act_args, (int, float)):
            act_args = [20.0 if act_args is None else float(act_args)] * count
        if len(activations) != count or len(act_args) != count:
            raise ArgumentError(f"need one activation / act_arg per layer ({count})")
        plans = [plan for _, plan in model.plans.layers]
        for i in range(1, count):
            if plans[i].q != plans[i - 1].r_dim:
                raise DimensionError(
                    f"layer {model.layer_names[i]!r} takes {plans[i].q} inputs but "
                    f"{model.layer_names[i - 1]!r} produces {plans[i - 1].r_dim}")
        self.names = model.layer_names
        self.mma = mma
        self.pipeline = pipeline
        self.codes = [_act_code(a) for a in activations]
        self.act_args = [float(a) for a in act_args]

        dev = device()
        staging = torch.empty(len(image), dtype=torch.uint8, pin_memory=True)
        staging.numpy()[:] = np.frombuffer(image, dtype=np.uint8)
        img = staging.to(dev, non_blocking=True)
        self.h2d_bytes = len(image)
        lib, st, base = _lib.lib(), stream_handle(), img.data_ptr()
        want16 = mma == "bf16"

        def unpack(offset, shape, code):
            out = torch.empty(shape, dtype=torch.float32, device=dev)
            out16 = torch.empty(shape, dtype=torch.bfloat16, device=dev) if want16 else None
            _lib.check(lib.dt_unpack_values(
                out.numel(), base + offset, _lib.DT_F64 if code == 1 else _lib.DT_F32,
                out.data_ptr(), out16.data_ptr() if out16 is not None else None, st))
            return out, out16

        self.factors, self.biases = [], []
        for rec, plan in zip(index, plans):
            xf, xf16 = unpack(rec.xf_offset, (plan.m, plan.rank), rec.dtype_code)
            wf, wf16 = unpack(rec.wf_offset, (plan.rank, plan.n), rec.dtype_code)
            bias, _ = unpack(rec.bias_offset, (rec.bias_len,), rec.dtype_code)
            if rec.bias_len != plan.r_dim:
                raise DimensionError(f"bias length {rec.bias_len} != output width {plan.r_dim}")
            self.factors.append(FactorPair.adopt(xf, wf, plan, (xf16, wf16) if want16 else None))
            self.biases.append(bias)
        torch.cuda.current_stream().synchronize()  # the image (and staging) can go now
        del img, staging
        self._ws = [None] * count
        # per-row-tile layer chaining (see forward): exact, but measured slower at config 3
        # (351 vs 323 us per forward: its clusters of 8 only launch on SMs the previous layer's
        # clusters free, which all finish within ~one tile of each other, and the x producer
        # then polls flags instead of a single grid dependency): off by default
        self.chain = False
        self._chain_key = None
        # fused layer chains (dt_chain_forward, k_tc_chain.cu): runs of reuse layers as ONE
        # kernel with the hidden activations kept in shared memory. Exact (bit-identical to the
        # layer-by-layer kernels) but measured slower at config 3 (314 vs ~213 us for layers
        # 1-6): a tile's six layers are a serial ~10 us-per-layer chain (phase A, cluster P
        # exchange, phase B + epilogue) that one tile in flight per cluster cannot hide, while
        # the per-layer kernel pipelines tiles. Opt-in.
        self.fuse = False

    @property
    def plans(self):
        return [fp.plan for fp in self.factors]

    def forward(self, x, out_dtype=torch.float32, graph: bool = False):
        """y = act_L(... act_1(x W_1 + b_1) ... W_L + b_L). Host (numpy) input returns a host
        array; a CUDA tensor returns a CUDA tensor (stream-ordered, no sync).

        graph=True (CUDA input): the layer chain is captured once per (input buffer, batch,
        dtypes) into a CUDA graph and replayed — one launch instead of ~25 us of host work per
        layer (what limits small per-GPU batches). The returned tensor is the graph's static
        output: the next graph forward on the same input buffer overwrites it."""
        if graph and isinstance(x, torch.Tensor) and x.is_cuda:
            return self._graph_forward(x, out_dtype)
        xt, host = as_device_matrix(x, name="input")
        if xt.shape[1] != self.factors[0].plan.q:
            raise DimensionError(f"input has {xt.shape[1]} columns, the first layer takes "
                                 f"{self.factors[0].plan.q}")
        code = _lib.DT_MMA_BF16 if self.mma == "bf16" else _lib.DT_MMA_FFMA
        mid = torch.bfloat16 if self.mma == "bf16" else torch.float32
        lib = _lib.lib()
        batch = xt.shape[0]
        last = len(self.factors) - 1
        # Row-tile layers with prepared operands chain on per-row-tile flags (dt_rows_chain):
        # layer i+1 loads rows layer i has finished while layer i still runs, so intermediate
        # activations rotate over three persistent buffers (a layer never overwrites rows an
        # earlier, still-running layer reads).
        ydt = lambda i: out_dtype if i == last else mid
        rows = [code == _lib.DT_MMA_BF16 and self.chain and
                fp.rows_prepared(b, c, _lib.DT_BF16 if ydt(i) == torch.bfloat16 else _lib.DT_F32)
                is not None and (i > 0 or xt.dtype == torch.bfloat16)
                for i, (fp, b, c) in enumerate(zip(self.factors, self.biases, self.codes))]
        bufs = flags = None
        if any(rows[i] and rows[i - 1] for i in range(1, last + 1)):
            bufs, flags = self._chain_state(batch, mid)
        runs = self._fused_runs(out_dtype) if (code == _lib.DT_MMA_BF16 and self.fuse and
                                               bufs is None) else {}
        with forward_pipeline(self.pipeline and self.mma == "bf16"):
            skip_to = 0
            for i, (fp, bias) in enumerate(zip(self.factors, self.biases)):
                if i < skip_to:
                    continue
                if i in runs and xt.dtype == torch.bfloat16 and xt.is_contiguous():
                    j = runs[i]
                    y = torch.empty((batch, self.factors[j].plan.r_dim), device=xt.device,
                                    dtype=torch.bfloat16)
                    self._run_chain(i, j, xt, y)
                    xt = y
                    skip_to = j + 1
                    continue
                need = lib.dt_forward_workspace_bytes(C.byref(_lib.plan_struct(fp.plan)), batch,
                                                      code)
                if self._ws[i] is None or self._ws[i].numel() < need:
                    self._ws[i] = torch.empty(max(need, 256), dtype=torch.uint8,
                                              device=xt.device)
                if bufs is not None and i < last:
                    y = bufs[(i + 1) % 3][: batch * fp.plan.r_dim].view(batch, fp.plan.r_dim)
                else:
                    y = torch.empty((batch, fp.plan.r_dim), device=xt.device, dtype=ydt(i))
                if bufs is not None and rows[i]:
                    wait = target = 0
                    if i > 0 and rows[i - 1]:
                        wait = flags[i - 1].data_ptr()
                        target = self._epoch * self._posts[i - 1]
                    post = flags[i].data_ptr() if i < last and rows[i + 1] else None
                    _lib.check(lib.dt_rows_chain(wait or None, target, post))
                forward_into(xt, fp, bias, self.codes[i], self.act_args[i], y, code,
                             ws=self._ws[i], cached=True)
                xt = y
        if bufs is not None:
            self._epoch += 1
        return xt.float().cpu().numpy() if host else xt

    def forward_host(self, hx, hy=None, *, chunks: int = 4, out_dtype=torch.bfloat16):
        """Pinned host x -> pinned host y with the copies overlapped: the batch is cut into
        `chunks` row blocks (multiples of 128 rows) and block i's host->device copy, forward
        (CUDA-graph replay on its own static buffers) and device->host copy run on three streams,
        so the PCIe transfers of one block hide the compute of its neighbours and the two copy
        directions run concurrently. Rows are independent (kernel.py:296-320 applied per row;
        the kernels' bits do not depend on the batch sharding), so the result equals
        forward(x). Returns hy (allocated pinned when None); synchronises before returning.

        hx: pinned CPU tensor (batch x q) of the dtype the first layer reads (bf16 on the
        tensor-core path)."""
        if not (isinstance(hx, torch.Tensor) and hx.device.type == "cpu" and hx.dim() == 2):
            raise ArgumentError("forward_host takes a 2-D CPU tensor (pinned for overlap)")
        if hx.shape[1] != self.factors[0].plan.q:
            raise DimensionError(f"input has {hx.shape[1]} columns, the first layer takes "
                                 f"{self.factors[0].plan.q}")
        batch, width = hx.shape[0], self.factors[-1].plan.r_dim
        if hy is None:
            hy = torch.empty((batch, width), dtype=out_dtype, pin_memory=True)
        if tuple(hy.shape) != (batch, width) or hy.dtype != out_dtype:
            raise DimensionError(f"output buffer must be {batch} x {width} {out_dtype}")
        if batch == 0:
            return hy
        per = -(-batch // max(1, chunks))
        per = -(-per // 128) * 128
        bounds = [(r, min(batch, r + per)) for r in range(0, batch, per)]
        key = (batch, hx.dtype, out_dtype, len(bounds))
        st = self.__dict__.get("_host_pipe")
        if st is None or st["key"] != key:
            dev = self.factors[0].xf.device
            st = {"key": key, "s_in": torch.cuda.Stream(), "s_out": torch.cuda.Stream(),
                  "xd": [torch.empty((b - a, hx.shape[1]), dtype=hx.dtype, device=dev)
                         for a, b in bounds],
                  "ev_in": [torch.cuda.Event() for _ in bounds],
                  "ev_c": [torch.cuda.Event() for _ in bounds],
                  "ev_out": [torch.cuda.Event() for _ in bounds]}
            self._host_pipe = st
        cur = torch.cuda.current_stream()
        st["s_in"].wait_stream(cur)
        for i, (a, b) in enumerate(bounds):
            with torch.cuda.stream(st["s_in"]):
                st["s_in"].wait_event(st["ev_c"][i])   # the previous call's forward read xd[i]
                st["xd"][i].copy_(hx[a:b], non_blocking=True)
                st["ev_in"][i].record()
            cur.wait_event(st["ev_in"][i])
            cur.wait_event(st["ev_out"][i])            # the graph's static output was copied out
            yd = self.forward(st["xd"][i], out_dtype=out_dtype, graph=True)
            st["ev_c"][i].record(cur)
            with torch.cuda.stream(st["s_out"]):
                st["s_out"].wait_event(st["ev_c"][i])
                hy[a:b].copy_(yd, non_blocking=True)
                st["ev_out"][i].record()
        st["s_out"].synchronize()
        return hy

    def _fused_runs(self, out_dtype):
        """{first: last} of the layer runs dt_chain_forward takes: >= 2 consecutive reuse layers
        on the row-tile kernel sharing n, rank and q/n, one elementwise activation on all but the
        last, the last identity (bf16 output, so the network's final layer only when out_dtype is
        bf16)."""
        key = ("runs", out_dtype)
        cache = self.__dict__.setdefault("_run_cache", {})
        if key in cache:
            return cache[key]
        lib = _lib.lib()
        last = len(self.factors) - 1
        sm, ident = _act_code("softmax"), _act_code("identity")

        def rows_ok(i):
            return lib.dt_rows_prepared_bytes(C.byref(_lib.plan_struct(self.factors[i].plan)),
                                              _lib.DT_BF16, _lib.DT_BF16) > 0

        runs, i = {}, 0
        while i <= last:
            best = None
            j = i + 1
            while j <= last and j - i < 8:
                hid = self.codes[i:j]
                if not (all(c == hid[0] for c in hid) and hid[0] not in (sm,)):
                    break
                # an identity head only: a softmax head runs on the row-tile kernel, whose fused
                # epilogue normalises the fp32 logits (the chain would store bf16 logits first)
                ends_ok = self.codes[j] == ident and (j < last or out_dtype == torch.bfloat16)
                plans = (_lib.Plan * (j - i + 1))(*[_lib.plan_struct(f.plan)
                                                   for f in self.factors[i:j + 1]])
                if ends_ok and all(rows_ok(k) for k in range(i, j + 1)) and \
                        lib.dt_chain_ok(plans, j - i + 1):
                    best = j
                j += 1
            if best is not None:
                runs[i] = best
                i = best + 1
            else:
                i += 1
        cache[key] = runs
        return runs

    def _run_chain(self, i, j, x, y):
        lib = _lib.lib()
        L = j - i + 1
        hidden = self.codes[i]
        ident = _act_code("identity")
        bufs = []
        for k in range(i, j + 1):
            act = hidden if k < j else ident
            buf = self.factors[k].rows_prepared(self.biases[k], act, _lib.DT_BF16)
            bufs.append(buf)
        plans = (_lib.Plan * L)(*[_lib.plan_struct(f.plan) for f in self.factors[i:j + 1]])
        ptrs = (C.c_void_p * L)(*[b.data_ptr() for b in bufs])
        _lib.check(lib.dt_chain_forward(plans, L, x.shape[0], x.data_ptr(), ptrs, hidden,
                                        self.act_args[i], self.codes[j], y.data_ptr(),
                                        stream_handle()))

    def _graph_forward(self, x, out_dtype):
        key = (x.data_ptr(), tuple(x.shape), x.dtype, out_dtype)
        graphs = self.__dict__.setdefault("_graphs", {})
        if key not in graphs:
            if len(graphs) >= 16:
                graphs.clear()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):  # warm-up: workspaces, prepared operands, modules
                self.forward(x, out_dtype)
            torch.cuda.current_stream().wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                y = self.forward(x, out_dtype)
            # the graph holds raw pointers into the workspaces (and chain buffers) it captured:
            # keep those tensors alive with it, so a later call that grows and replaces a
            # workspace cannot hand the old memory to the allocator while the graph may replay
            refs = [w for w in self._ws if w is not None] + list(self.__dict__.get("_bufs", []))
            refs += list(self.__dict__.get("_flags", []))
            graphs[key] = (g, y, refs)
        g, y, _ = graphs[key]
        g.replay()
        return y

    def _chain_state(self, batch, mid):
        """Three rotating activation buffers and per-layer tile flags for this batch size."""
        key = (batch, mid)
        if self._chain_key != key:
            width = max(fp.plan.r_dim for fp in self.factors)
            dev = self.factors[0].xf.device
            self._bufs = [torch.empty(batch * width, dtype=mid, device=dev) for _ in range(3)]
            tiles = -(-batch // 128)
            self._flags = [torch.zeros(tiles, dtype=torch.int32, device=dev) for _ in self.factors]
            self._posts = [_lib.lib().dt_rows_posts_per_tile(C.byref(_lib.plan_struct(fp.plan)))
                           for fp in self.factors]
            self._epoch = 1
            self._chain_key = key
        return self._bufs, self._flags

    __call__ = forward
