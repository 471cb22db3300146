"""Training harness around the GoCkpt hot path (NOT the method; used by bench.py).

  Gpt2GemmStandIn  the forward/backward stand-in: every GEMM of a GPT-2 small
                   training step (12 layers, d=768, 12 heads, seq 1024, vocab
                   50257 padded to 50304 as GPT-2 trainers do so cuBLAS can use
                   its aligned sm_100 kernels; fwd + dgrad + wgrad, attention as
                   batched GEMMs) on
                   fixed random bf16 operands, captured once in a CUDA graph.
                   cuBLAS library GEMMs: they stand for the step the checkpoint
                   overlaps, they are not part of the checkpoint path.
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


class Gpt2GemmStandIn:
    def __init__(self, tokens: int = 16 * 1024, d: int = 768, layers: int = 12, heads: int = 12,
                 seq: int = 1024, vocab: int = 50304, device="cuda", seed: int = 0):
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        bf = torch.bfloat16
        self.flops = 0
        self.ops = []  # (kind, A, B, C, dA, dB)
        T, B = tokens, tokens // seq

        def rnd(*shape):
            return (torch.randn(*shape, generator=g, device=device, dtype=torch.float32) * 0.02).to(bf)

        def gemm(M, K, N):
            A, Bm = rnd(M, K), rnd(K, N)
            C = torch.empty(M, N, device=device, dtype=bf)
            self.ops.append(("mm", A, Bm, C, torch.empty_like(A), torch.empty_like(Bm)))
            self.flops += 3 * 2 * M * K * N

        def bgemm(Bt, M, K, N):
            A, Bm = rnd(Bt, M, K), rnd(Bt, K, N)
            C = torch.empty(Bt, M, N, device=device, dtype=bf)
            self.ops.append(("bmm", A, Bm, C, torch.empty_like(A), torch.empty_like(Bm)))
            self.flops += 3 * 2 * Bt * M * K * N

        hd = d // heads
        for _ in range(layers):
            gemm(T, d, 3 * d)                  # qkv
            bgemm(B * heads, seq, hd, seq)     # q k^T
            bgemm(B * heads, seq, seq, hd)     # p v
            gemm(T, d, d)                      # attn out
            gemm(T, d, 4 * d)                  # fc
            gemm(T, 4 * d, d)                  # proj
        gemm(T, d, vocab)                      # lm head
        self.graph = None
        self.tokens = tokens

    def _run(self):
        for kind, A, Bm, C, dA, dB in self.ops:       # forward
            (torch.mm if kind == "mm" else torch.bmm)(A, Bm, out=C)
        for kind, A, Bm, C, dA, dB in reversed(self.ops):  # backward: dgrad + wgrad
            if kind == "mm":
                torch.mm(C, Bm.t(), out=dA)
                torch.mm(A.t(), C, out=dB)
            else:
                torch.bmm(C, Bm.transpose(1, 2), out=dA)
                torch.bmm(A.transpose(1, 2), C, out=dB)

    def capture(self):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                self._run()
        torch.cuda.current_stream().wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._run()
        torch.cuda.synchronize()

    def __call__(self):
        if self.graph is None:
            self._run()
        else:
            self.graph.replay()


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
