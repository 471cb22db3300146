"""Training harness around the GoCkpt hot path (NOT the method; used by bench.py).

  TransformerGemmStandIn  the forward/backward stand-in: every GEMM of a
                   GPT-2 small / Llama-2 7B / 13B training step (fwd + dgrad +
                   wgrad, attention as batched GEMMs; GPT-2's vocab padded to
                   50304 as GPT-2 trainers do so cuBLAS can use its aligned
                   sm_100 kernels) on fixed random bf16 operands, captured once
                   in a CUDA graph. cuBLAS library GEMMs: they stand for the step
                   the checkpoint overlaps, they are not part of the checkpoint path.
  ClockSampler     nvidia-smi clocks / throttle reasons during the timed region.
  dist helpers     ZeRO-1 plumbing: every rank derives the same session schedule
                   from the global step (no communication on the checkpoint
                   path); timings are maxed over ranks.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import tempfile

import torch


MODELS = {
    # name: (params, d, layers, heads, ffn, vocab, gated-MLP, seq); vocab padded to a multiple of 64
    "gpt2-small": (124_439_808, 768, 12, 12, 3072, 50304, False, 1024),
    "llama2-7b": (6_738_415_616, 4096, 32, 32, 11008, 32000, True, 4096),
    "llama2-13b": (13_015_864_320, 5120, 40, 40, 13824, 32000, True, 4096),
}
FLAT_1M = 1 << 20  # BASELINE config 1: a flat fp32 vector, F/B = a spin kernel (SpinStandIn)


def standin_shapes(model: str, tokens: int):
    """The GEMMs of one decoder-only training step of `model` on `tokens` tokens: a list of
    (kind, shape, repeat) with kind "mm" (M, K, N) or "bmm" (batch, M, K, N), forward order."""
    _, d, layers, heads, ffn, vocab, gated, mseq = MODELS[model]
    seq = min(mseq, tokens)
    T, B = tokens, max(1, tokens // seq)
    hd = d // heads
    return [("mm", (T, d, 3 * d), layers),                      # qkv
            ("bmm", (B * heads, seq, hd, seq), layers),          # q k^T
            ("bmm", (B * heads, seq, seq, hd), layers),          # p v
            ("mm", (T, d, d), layers),                          # attn out
            ("mm", (T, d, (2 if gated else 1) * ffn), layers),  # fc (gate+up when gated)
            ("mm", (T, ffn, d), layers),                        # down / proj
            ("mm", (T, d, vocab), 1)]                           # lm head


def standin_flops(model: str, tokens: int) -> int:
    """FLOPs of one stand-in step (forward + dgrad + wgrad = 3 x 2MKN per GEMM); host-only."""
    f = 0
    for kind, sh, rep in standin_shapes(model, tokens):
        M, K, N = sh[-3:]
        f += rep * 3 * 2 * M * K * N * (sh[0] if kind == "bmm" else 1)
    return f


class TransformerGemmStandIn:
    """Every GEMM of one decoder-only transformer training step (forward, dgrad, wgrad) on
    fixed random bf16 operands, in CUDA graphs: the F/B the checkpoint overlaps (harness).

    Shapes follow the named model (standin_shapes); attention score/value products are batched
    GEMMs over heads. Layers share one set of operand buffers (same FLOPs and shapes,
    1/layers of the memory). cuBLAS library GEMMs, not part of the checkpoint path.
    capture(bwd_parts=P) splits the backward into P graphs (each op's layer repeats divided
    evenly), so gradient buckets can be reduce-scattered while the rest of the backward runs.
    """

    def __init__(self, model: str = "gpt2-small", tokens: int = 16 * 1024, device="cuda", seed: int = 0):
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        bf = torch.bfloat16
        self.ops = []  # (kind, A, B, C, dA, dB, repeat)
        self.model, self.tokens = model, tokens
        self.flops = standin_flops(model, tokens)

        def rnd(*shape):
            return (torch.randn(*shape, generator=g, device=device, dtype=torch.float32) * 0.02).to(bf)

        for kind, sh, rep in standin_shapes(model, tokens):
            if kind == "mm":
                M, K, N = sh
                A, Bm, C = rnd(M, K), rnd(K, N), torch.empty(M, N, device=device, dtype=bf)
            else:
                Bt, M, K, N = sh
                A, Bm, C = rnd(Bt, M, K), rnd(Bt, K, N), torch.empty(Bt, M, N, device=device, dtype=bf)
            self.ops.append((kind, A, Bm, C, torch.empty_like(A), torch.empty_like(Bm), rep))
        self.graphs = None
        self.bwd_parts = 1

    def _forward(self):
        for kind, A, Bm, C, dA, dB, rep in self.ops:
            for _ in range(rep):
                (torch.mm if kind == "mm" else torch.bmm)(A, Bm, out=C)

    def _backward(self, part: int = 0, parts: int = 1):
        for kind, A, Bm, C, dA, dB, rep in reversed(self.ops):   # dgrad + wgrad, last layer first
            for _ in range(rep * part // parts, rep * (part + 1) // parts):
                if kind == "mm":
                    torch.mm(C, Bm.t(), out=dA)
                    torch.mm(A.t(), C, out=dB)
                else:
                    torch.bmm(C, Bm.transpose(1, 2), out=dA)
                    torch.bmm(A.transpose(1, 2), C, out=dB)

    def _run(self):
        self._forward()
        for k in range(self.bwd_parts):
            self._backward(k, self.bwd_parts)

    def capture(self, bwd_parts: int = 1):
        self.bwd_parts = max(1, bwd_parts)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                self._run()
        torch.cuda.current_stream().wait_stream(s)
        self.graphs = []
        for k in range(-1, self.bwd_parts):
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph):
                if k < 0:
                    self._forward()
                else:
                    self._backward(k, self.bwd_parts)
            self.graphs.append(gph)
        torch.cuda.synchronize()

    def forward(self):
        if self.graphs is None:
            self._forward()
        else:
            self.graphs[0].replay()

    def backward(self, part: int):
        if self.graphs is None:
            self._backward(part, self.bwd_parts)
        else:
            self.graphs[1 + part].replay()

    def __call__(self):
        self.forward()
        for k in range(self.bwd_parts):
            self.backward(k)


class SpinStandIn:
    """A fixed-duration F/B stand-in (BASELINE config 1: "spin kernel 1 ms (and 0)"): one
    torch.cuda._sleep spin kernel of `ms` at the device's clock; ms = 0 launches nothing."""

    def __init__(self, ms: float, device="cuda"):
        self.ms = ms
        self.flops = 0
        self.bwd_parts = 1
        rate_khz = torch.cuda.get_device_properties(device).clock_rate if ms > 0 else 0
        self.cycles = int(ms * rate_khz)  # kHz x ms = cycles

    def capture(self, bwd_parts: int = 1):
        pass

    def forward(self):
        if self.cycles:
            torch.cuda._sleep(self.cycles)

    def backward(self, part: int):
        pass

    def __call__(self):
        self.forward()


def rs_buckets(n: int, world: int, bucket_bytes: int = 512 << 20, align: int = 512):
    """ZeRO-1 gradient reduce-scatter buckets: (offset, count) ranges of the rank's n-element shard,
    each the output of one reduce_scatter_tensor whose input (world x count bf16, laid out
    contiguously per bucket) is about bucket_bytes. Covers [0, n) in order."""
    cnt = max(align, (bucket_bytes // (2 * world)) // align * align)
    return [(o, min(cnt, n - o)) for o in range(0, n, cnt)]


def Gpt2GemmStandIn(tokens: int = 16 * 1024, device="cuda", seed: int = 0):
    return TransformerGemmStandIn("gpt2-small", tokens, device, seed)


class ClockSampler:
    """nvidia-smi --query-gpu ... -lms 200 in the background (the B200 profiling recipe's clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int = 0):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        if not shutil.which("nvidia-smi"):
            return self
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        self.fh = open(self.path, "w")
        self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits", "-lms", "200"],
                                     stdout=self.fh, stderr=subprocess.DEVNULL)
        return self

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax.append(float(parts[2]))
                    power.append(float(parts[3]))
                except ValueError:
                    continue
                for nm, val in zip(names, parts[5:9]):
                    if val.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = sorted(x for x, p in zip(sm, power) if p > 250) or sorted(sm)
        return {"sm_mhz": loaded[len(loaded) // 2], "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power)}


def session_part(step_in_interval: int, K: int) -> int:
    """Session schedule inside a checkpoint interval: steps 1..K of the interval are parts 1..K.

    Every rank evaluates it on the global step, so all ranks' sessions target the
    same version T = t0 + K - 1 without any communication.
    """
    return step_in_interval if 1 <= step_in_interval <= K else 0


def max_over_ranks(x: float) -> float:
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return x
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_ranks_ok(ok: bool) -> bool:
    """Global checkpoint commit: complete only when every rank finalized (P:372 'Rank 0 monitoring')."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return ok
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def zero1_shard(n_total: int, world: int, rank: int, align: int = 1024):
    """ZeRO-1 flat-buffer shard: pad to a multiple of world*align, rank r owns [r*n_r, (r+1)*n_r)."""
    unit = world * align
    padded = (n_total + unit - 1) // unit * unit
    n_r = padded // world
    return rank * n_r, n_r, padded


def commit_global(directory: str, step: int, local_ok: bool, files: list[str] | None = None,
                  n_total: int | None = None, n_per_rank: int | None = None, align: int | None = None) -> bool:
    """Global checkpoint commit ("Rank 0 monitoring completion by other Ranks"): every rank
    reports whether its shard's file is durable; rank 0 writes MANIFEST.json (atomic rename) only
    if all did. Returns whether the global checkpoint is complete."""
    import json
    import torch.distributed as dist
    ok = all_ranks_ok(local_ok)
    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_available() and dist.is_initialized() else 0
    if ok and rank == 0:
        man = {"step": step, "world": world,
               "files": files or [f"ckpt_{step}.rank{r}.bin" for r in range(world)],
               "n_total": n_total, "n_per_rank": n_per_rank, "align": align}
        tmp = os.path.join(directory, "MANIFEST.json.tmp")
        with open(tmp, "w") as fh:
            json.dump(man, fh)
            fh.flush()
            os.fsync(fh.fileno())
        os.replace(tmp, os.path.join(directory, "MANIFEST.json"))
    return ok


def load_resharded(directory: str, world_new: int, rank_new: int, align: int | None = None):
    """Load rank `rank_new`'s ZeRO-1 shard for a new data-parallel degree `world_new` from a global
    checkpoint written at another degree (MANIFEST.json): the new rank's range [r'n', (r'+1)n') of
    the flat buffer is read from the old ranks' files with gck_load_checkpoint_range (every
    touched block CRC-verified). P:376: "during loading, these shards are fetched". Positions past
    the model's n_total (ZeRO padding) are zero. Returns (master, m, v, step)."""
    import json
    import numpy as np
    from . import gockpt as G
    man = json.load(open(os.path.join(directory, "MANIFEST.json")))
    N, W, n_old = man["n_total"], man["world"], man["n_per_rank"]
    off, n_new, _ = zero1_shard(N, world_new, rank_new, align or man.get("align") or 1024)
    out = [np.zeros(n_new, np.float32) for _ in range(3)]
    step = None
    for r in range(W):
        o0 = r * n_old
        lo, hi = max(off, o0), min(off + n_new, o0 + n_old, N)
        if lo >= hi:
            continue
        views = [x[lo - off:hi - off] for x in out]
        _, _, _, h = G.load_checkpoint_range(os.path.join(directory, man["files"][r]), lo - o0, hi - lo, views)
        if step is not None and h["step"] != step:
            raise ValueError("shards of different steps in one manifest")
        step = h["step"]
    return out[0], out[1], out[2], step
