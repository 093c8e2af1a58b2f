"""Multi-GPU evaluation of one encrypted input ("Out-P").

The reference only *models* output parallelism analytically
(`costs.py:80-88`, the paper's "Out 16-P / Out Full-P").
Here it executes: each block's output units (dense rows / conv output
channels) are partitioned across ranks, every rank builds the block's
shared input sum itself (replicated — it is ~1% of a layer's gates), runs
its units on its own GPU, and the layer's output ciphertexts are all-gathered
(torch.distributed: NCCL between GPUs, gloo in the CPU tests) before the next
block.  Gates never cross ranks inside a layer, so the only exchange is one
all-gather of p x 2,524 B per layer.
"""

from __future__ import annotations

import numpy as np

from hebnn.circuits import CipherWord
from hebnn.compiler import EvalOptions, eval_model
from hebnn.model import BatchNorm, ConvLayer, DenseLayer, SignActivation, TernaryModel, model_blocks


def partition(count, world, costs=None):
    """Contiguous split of `count` output units over `world` ranks: equal unit
    counts, or — with per-unit `costs` (e.g. gates per neuron) — equal cost
    (cfg4's ternary rows have very different DAG sizes)."""
    if costs is None:
        bounds = [round(r * count / world) for r in range(world + 1)]
        return [(bounds[r], bounds[r + 1]) for r in range(world)]
    costs = [max(0.0, float(c)) for c in costs]
    total = sum(costs) or 1.0
    bounds, acc, r = [0], 0.0, 1
    for i, c in enumerate(costs):
        acc += c
        while r < world and acc >= r * total / world:
            bounds.append(i + 1)
            r += 1
    while len(bounds) < world + 1:
        bounds.append(count)
    bounds[-1] = count
    return [(bounds[k], max(bounds[k], bounds[k + 1])) for k in range(world)]


def unit_costs(block, options=EvalOptions()):
    """Predicted encrypted additions per output unit (compiler.plan_row), a
    proxy for its gate count."""
    from hebnn.compiler import plan_row
    from hebnn.model import flat_filter

    lin = block.linear
    rows = lin.weights if isinstance(lin, DenseLayer) else [tuple(flat_filter(f)) for f in lin.filters]
    return [plan_row(r, None, options).predicted_adds + 1 for r in rows]


def _sub_block_model(block, lo, hi, output_mode, is_last):
    """A one-block TernaryModel computing output units [lo, hi) of `block`."""
    lin = block.linear
    if isinstance(lin, DenseLayer):
        mags = lin.magnitudes[lo:hi] if lin.magnitudes is not None else None
        sub = DenseLayer(tuple(lin.weights[lo:hi]), tuple(lin.bias[lo:hi]), magnitudes=mags)
    else:
        mags = lin.magnitudes[lo:hi] if lin.magnitudes is not None else None
        sub = ConvLayer(tuple(lin.filters[lo:hi]), tuple(lin.bias[lo:hi]), stride=lin.stride, magnitudes=mags)
    layers = [sub]
    if block.bn is not None:
        bn = block.bn
        layers.append(BatchNorm(bn.gamma[lo:hi], bn.beta[lo:hi], bn.mu[lo:hi], bn.sigma2[lo:hi], bn.epsilon))
    mode = output_mode if is_last else "sign_bits"
    if mode == "sign_bits":
        layers.append(SignActivation())
    return TernaryModel(block.in_shape, tuple(layers), mode)


def _units(block):
    lin = block.linear
    return len(lin.weights) if isinstance(lin, DenseLayer) else len(lin.filters)


def _per_unit(block):
    """Output bits per output unit (conv: one per window position)."""
    if isinstance(block.linear, DenseLayer):
        return 1
    _, oh, ow = block.out_shape
    return oh * ow


class OutPEvaluator:
    """Evaluate a model on encrypted inputs with layer-wise output partitioning.

    ctx_factory(): returns a fresh GateBackend-compatible context with
    `import_ciphertexts` / `export_ciphertexts` (TfheContext) on this rank's
    device.  comm: object with `rank`, `world` and `all_gather(np.ndarray) ->
    list[np.ndarray]` (see `TorchComm`).
    """

    def __init__(self, ctx_factory, comm, options=EvalOptions(), balance="gates"):
        self.ctx_factory = ctx_factory
        self.comm = comm
        self.options = options
        self.balance = balance  # "gates" (predicted cost) or "units"
        self.stats = []

    def run(self, model, input_cts):
        """input_cts: [d][lanes][n+1] uint32 encrypted input bits (identical on
        every rank).  Returns the final layer's output ciphertexts in unit
        order, gathered on every rank: a list with one [lanes][n+1] array per
        bit (sign_bits) or per word a list of bit arrays plus signedness."""
        cts = np.asarray(input_cts, np.uint32)
        blocks = model_blocks(model, stride=self.options.stride)
        result = None
        for bi, block in enumerate(blocks):
            is_last = bi == len(blocks) - 1
            costs = unit_costs(block, self.options) if self.balance == "gates" else None
            lo, hi = partition(_units(block), self.comm.world, costs)[self.comm.rank]
            ctx = self.ctx_factory()
            dev_path = getattr(self.comm, "device_tensors", False) and hasattr(ctx, "import_ciphertexts_device")
            x = ctx.import_ciphertexts_device(cts) if dev_path and not isinstance(cts, np.ndarray) \
                else ctx.import_ciphertexts(self._host(cts))
            outs = []
            if hi > lo:
                sub = _sub_block_model(block, lo, hi, model.output_mode, is_last)
                outs, _ = eval_model(ctx, sub, x, self.options)
            if is_last and model.output_mode == "score_words":
                # words: gather (bits, width, signed) per unit
                flat = [b for w in outs for b in w.bits]
                widths = np.array([w.width for w in outs] + [0], np.int64)[:-1]
                signed = np.array([int(w.signed) for w in outs], np.int64)
                if dev_path:  # word bits gathered as device tensors (NCCL), read once at the end
                    import torch

                    local = ctx.export_ciphertexts_device(flat) if flat else torch.zeros(
                        (0, ctx.lanes, ctx.params.n + 1), dtype=torch.int32, device=f"cuda:{ctx.device}")
                    all_cts = [t.cpu().numpy().view(np.uint32) for t in self.comm.all_gather_tensor(local)]
                else:
                    local = ctx.export_ciphertexts(flat) if flat else np.zeros((0, ctx.lanes, ctx.params.n + 1),
                                                                               np.uint32)
                    all_cts = self.comm.all_gather(local)
                all_w = self.comm.all_gather(widths)
                all_s = self.comm.all_gather(signed)
                result = []
                for cts_r, w_r, s_r in zip(all_cts, all_w, all_s):
                    off = 0
                    for w, sg in zip(w_r, s_r):
                        result.append((cts_r[off:off + w], bool(sg)))
                        off += w
            elif dev_path:  # NCCL all-gather of device-resident ciphertexts (no host staging)
                import torch

                local = ctx.export_ciphertexts_device(outs) if outs else \
                    torch.zeros((0, ctx.lanes, ctx.params.n + 1), dtype=torch.int32, device=f"cuda:{ctx.device}")
                cts = torch.cat(self.comm.all_gather_tensor(local), dim=0)
                result = [c.cpu().numpy().view(np.uint32) for c in cts] if is_last else None
            else:
                local = ctx.export_ciphertexts(outs) if outs else np.zeros((0, ctx.lanes, ctx.params.n + 1), np.uint32)
                gathered = self.comm.all_gather(local)
                cts = np.concatenate(gathered, axis=0)
                result = list(cts)
            # after the export: its flush ran the block's remaining gates
            self.stats.append({"block": bi, "units": (lo, hi), "counted_gates": ctx.gate_count,
                               "executed": dict(ctx.exec_stats)})
        return result

    @staticmethod
    def _host(cts):
        if isinstance(cts, np.ndarray):
            return cts
        return cts.cpu().numpy().view(np.uint32)


class TorchComm:
    """all-gather of variable-length uint32 arrays over torch.distributed; with
    NCCL (device_tensors) layer outputs are gathered as CUDA tensors straight
    from and into the engine pools (hb_pool_gather_device / hb_pool_put_device)."""

    def __init__(self, device=None):
        import torch
        import torch.distributed as dist

        self.torch = torch
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device if device is not None else ("cuda" if dist.get_backend() == "nccl" else "cpu")
        self.device_tensors = str(self.device).startswith("cuda")

    def all_gather_tensor(self, t):
        """all-gather of a device tensor with a variable leading dimension."""
        torch, dist = self.torch, self.dist
        lead = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        sizes = [torch.zeros_like(lead) for _ in range(self.world)]
        dist.all_gather(sizes, lead)
        sizes = [int(v.item()) for v in sizes]
        mx = max(sizes) if sizes else 0
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        bufs = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(bufs, pad)
        torch.cuda.synchronize(t.device)
        return [b[:n] for b, n in zip(bufs, sizes)]

    def all_gather(self, arr):
        torch, dist = self.torch, self.dist
        arr = np.ascontiguousarray(arr)
        shape = list(arr.shape)
        lead = torch.tensor([shape[0] if shape else 0], dtype=torch.int64, device=self.device)
        sizes = [torch.zeros_like(lead) for _ in range(self.world)]
        dist.all_gather(sizes, lead)
        sizes = [int(s.item()) for s in sizes]
        inner = shape[1:]
        per = int(np.prod(inner)) if inner else 1
        mx = max(sizes) if sizes else 0
        flat = np.zeros(mx * per, dtype=np.int64 if arr.dtype != np.uint32 else np.int32)
        src = arr.reshape(-1).view(np.int32) if arr.dtype == np.uint32 else arr.reshape(-1).astype(np.int64)
        flat[: src.size] = src
        t = torch.from_numpy(flat).to(self.device)
        bufs = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(bufs, t)
        out = []
        for s, b in zip(sizes, bufs):
            v = b.cpu().numpy()[: s * per]
            v = v.view(np.uint32) if arr.dtype == np.uint32 else v.astype(arr.dtype)
            out.append(v.reshape([s] + inner))
        return out


def decode_scores(ctx, words):
    """Decrypt gathered score words [(bits [w][lanes][n+1], signed)] -> ints [lanes][units]."""
    vals = []
    for bits_cts, signed in words:
        bits = ctx.keys.decrypt(bits_cts.reshape(-1, bits_cts.shape[-1])).reshape(bits_cts.shape[:2])
        w = bits.shape[0]
        v = (bits.astype(np.int64) << np.arange(w)[:, None]).sum(axis=0)
        if signed:
            v = np.where(v >= 1 << (w - 1), v - (1 << w), v)
        vals.append(v)
    return np.stack(vals, axis=1)


__all__ = ["OutPEvaluator", "TorchComm", "partition", "decode_scores", "CipherWord"]
