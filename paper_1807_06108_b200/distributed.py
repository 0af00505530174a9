"""Multi-GPU sharding of the sampled-trajectory core: one process per GPU.

Samples shard naturally: rank r rolls out its own K_local
samples with GLOBAL sample indices in the Philox counter
(sample_offset = r * K_local), so the noise of a sharded run is exactly the
noise of one big run.  Per MPC iteration the only exchange is one all_gather
of each rank's weighting record (rho_r, Z_r, sum w^2_r, n_finite_r,
N_r[T*m]; 4 + T*m doubles, 3.2 KB at config 3) over NCCL; every rank then
merges the records in rank order with the same log-sum-exp rescale
exp(-(rho_r - rho)/lambda) (the finalize kernel) and applies the identical
update, plant step and shift -- one collective instead of a MIN all-reduce
followed by a SUM all-reduce.

Sharding (`scaling`): "weak" -- K samples per GPU (rank r owns global samples
[r K, (r+1) K)); "strong" -- BASELINE config 3's K/N split of a fixed global K
(shard_strong: ragged when N does not divide K, the first K mod N ranks one
sample more).

Two transports for the exchange:
  "nccl" (default) -- a reduce kernel merges the rank's CTA records into one,
         all_gather_into_tensor gathers the `world` records, the finalize
         merges them: three kernels of ours plus the collective per step;
  "p2p"  (JM_EXCHANGE=p2p) -- no collective library on the data path: each
         rank owns a symmetric buffer (torch.distributed._symmetric_memory,
         peer pointers over NVLink/NVSwitch); the rollout kernel's CTAs store
         their records straight into every rank's buffer and raise epoch flags
         there (system-scope release), the finalize waits on its own flags on
         the device (jm_loop_rollout_push / jm_loop_finish_peers) -- the step
         never returns to the host or a collective launch.  Two forms: flat
         (world < 6: every rank merges world x grid CTA records) and two-level
         (world >= 6 or strong scaling, `two_level`; JM_P2P_TWO_LEVEL=0/1
         overrides: a reduce kernel pushes one record per rank -- the NCCL
         transport's merge tree, bit for bit).  It has run at world 1 only
         (this pod exposes one GPU), hence not the default.
Every rank agrees on the transport before the first step (an all_reduce of
each rank's setup result), so a rank whose peer-buffer setup failed cannot
leave the others waiting in a different exchange.

torch.distributed is the plumbing (process group, rendezvous of the symmetric
buffers, streams); all arithmetic is in libjmppi.so.  The host-side logic here
(shard ranges, record exchange, rank-order merge) is covered on CPU by
tests/test_distributed.py with world_size 2 over gloo.
"""

from __future__ import annotations

import ctypes as C
import os
import sys
from dataclasses import dataclass
from typing import Tuple

import numpy as np

from . import _lib as L
from . import engine


def shard(k_per_rank: int, rank: int) -> Tuple[int, int]:
    """(sample_offset, count) of a rank under weak scaling (K_local fixed per GPU)."""
    return rank * k_per_rank, k_per_rank


def shard_for(scaling: str, k: int, rank: int, world: int) -> Tuple[int, int]:
    """(sample_offset, count): weak -- k samples per rank; strong -- k in total."""
    if scaling == "weak":
        return shard(k, rank)
    if scaling == "strong":
        return shard_strong(k, rank, world)
    raise ValueError(f"scaling must be weak or strong, got {scaling!r}")


def shard_strong(k_total: int, rank: int, world: int) -> Tuple[int, int]:
    """(sample_offset, count) when a fixed global K is split over `world` ranks."""
    base, rem = divmod(k_total, world)
    count = base + (1 if rank < rem else 0)
    offset = rank * base + min(rank, rem)
    return offset, count


def agree(ok: bool, group=None) -> bool:
    """True iff `ok` on every rank (an all_reduce MIN of a flag; CPU tensor under gloo)."""
    import torch
    import torch.distributed as dist

    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return bool(t.item())


def exchange_records(local, group=None):
    """All-gather one record per rank into a (world, rec) tensor, rank order.

    Uses all_gather_into_tensor where the backend has it (NCCL) and the list
    form otherwise (gloo on CPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    if local.is_cuda:
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    else:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local.contiguous(), group=group)
        out = torch.stack(parts)
    return out


TWO_LEVEL_MIN_WORLD = 6


def use_two_level(world: int, env=None) -> bool:
    """Whether the p2p exchange reduces each rank's CTA records to one before
    the push: from TWO_LEVEL_MIN_WORLD ranks, unless JM_P2P_TWO_LEVEL=0/1 says."""
    env = os.environ if env is None else env
    v = env.get("JM_P2P_TWO_LEVEL", "")
    if v not in ("", "0", "1"):
        raise ValueError(f"JM_P2P_TWO_LEVEL must be 0 or 1, got {v!r}")
    return bool(int(v)) if v else world >= TWO_LEVEL_MIN_WORLD


@dataclass
class ShardedLoop:
    """Closed-loop MPC with the sample set sharded over the ranks of a process group.

    Every rank holds an identical plant state (same seed, same merged update),
    so the trajectory equals a single-GPU run over rank-count x K_local samples
    up to the reduction order of the merge."""

    ctx: object
    world: int
    rank: int
    group: object = None
    transport: str = "nccl"
    two_level: bool = None  # p2p only; None: use_two_level(world) (always two-level under strong scaling)
    scaling: str = "weak"
    k_total: int = 0
    nccl_graph: object = None  # NCCL transport: the captured step (None: not tried yet; False: direct enqueue)

    @classmethod
    def create(cls, task, cfg, rank: int, world: int, device: int, precision=None, group=None, transport="nccl",
               scaling="weak"):
        off, cnt = shard_for(scaling, cfg.samples_m, rank, world)
        ctx = engine.get_context(task.model, task.cost_model, cfg, samples=cnt, precision=precision,
                                 sample_offset=off, device=device)
        k_total = cfg.samples_m if scaling == "strong" else world * cfg.samples_m
        # (ragged strong shards may differ in their CTA grids: one record per rank)
        return cls(ctx, world, rank, group, transport, True if scaling == "strong" else None, scaling, k_total)

    def launches_per_step(self) -> int:
        """Kernels of ours per control step (the NCCL collective not counted)."""
        if self.transport == "p2p":
            return 3 if self.two_level else 2
        return 3  # rollout, reduce, finalize

    def init(self, x0, u_init, seed: int, max_steps: int):
        import torch

        lib, h = self.ctx.lib, self.ctx.h
        x0 = np.ascontiguousarray(x0, float)
        ui = np.ascontiguousarray(u_init, float)
        self.ctx.check(lib.jm_loop_init(h, L.dptr(x0), L.dptr(ui), C.c_uint64(seed), C.c_uint64(0), max_steps))
        rs = C.c_int64()
        self.ctx.check(lib.jm_record_doubles(h, C.byref(rs)))
        dev = torch.device("cuda", self.ctx.device)
        # one explicit (non-legacy) stream carries the kernels AND the collective:
        # torch's default stream is the legacy stream 0, which jm_set_stream
        # would read as "the context's own non-blocking stream"
        self.stream = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(self.stream):
            self.record = torch.zeros(rs.value, dtype=torch.float64, device=dev)
        self.ctx.check(lib.jm_set_stream(h, C.c_void_p(self.stream.cuda_stream)))
        torch.cuda.synchronize(dev)
        if self.transport == "p2p":
            if self.two_level is None:
                self.two_level = use_two_level(self.world)  # (a bad JM_P2P_TWO_LEVEL raises on every rank)
            buf, err = None, None
            try:  # the local half of the setup: the symmetric allocation
                buf = self._alloc_peers(dev)
            except (RuntimeError, OSError, ImportError, AttributeError) as exc:
                err = exc
            # every rank takes the same transport: p2p only if it could be set up everywhere
            if agree(err is None, self.group):
                self._init_peers(dev, buf)
            else:
                self.transport = "nccl"
                self.p2p_error = err

    def _alloc_peers(self, dev):
        import torch
        import torch.distributed._symmetric_memory as symm

        n = int(self.ctx.lib.jm_peer_buffer_doubles(self.ctx.h, self.world))
        buf = symm.empty(n, dtype=torch.float64, device=dev)
        buf.zero_()  # epoch flags start at 0
        torch.cuda.synchronize(dev)
        return buf

    def _init_peers(self, dev, buf):
        """Rendezvous of the symmetric exchange buffers + their peer addresses (jm_peer_buffer_doubles layout)."""
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        lib, h = self.ctx.lib, self.ctx.h
        hdl = symm.rendezvous(buf, self.group if self.group is not None else dist.group.WORLD)
        ptrs = [int(p) for p in hdl.buffer_ptrs]
        off = buf.data_ptr() - ptrs[self.rank]  # the same offset in every rank's symmetric allocation
        self.peer_bases = torch.tensor([p + off for p in ptrs], dtype=torch.int64, device=dev)
        self.peer_buf, self.symm_handle = buf, hdl
        torch.cuda.synchronize(dev)
        dist.barrier(group=self.group)  # every rank's flags are zero before anyone pushes
        # the whole step is device-side (no collective, no host wait): one CUDA
        # graph of its two (flat) or three (two-level) kernels, replayed per control step
        lib, h = self.ctx.lib, self.ctx.h
        self.graph = torch.cuda.CUDAGraph()
        if self.two_level:
            push, finish = lib.jm_loop_rollout_reduce_push, lib.jm_loop_finish_reduced_peers
        else:
            push, finish = lib.jm_loop_rollout_push, lib.jm_loop_finish_peers
        with torch.cuda.graph(self.graph, stream=self.stream):
            self.ctx.check(push(h, C.c_void_p(self.peer_bases.data_ptr()), self.rank, self.world))
            self.ctx.check(finish(h, C.c_void_p(self.peer_buf.data_ptr()), self.world))

    def step(self):
        """One control step: local rollout + record, exchange, merge/update/plant/shift."""
        import torch

        lib, h = self.ctx.lib, self.ctx.h
        with torch.cuda.stream(self.stream):
            if self.transport == "p2p":
                self.graph.replay()
                return
            if self.nccl_graph is None:
                if self._capture_nccl_step():
                    return  # (the capture's eager step was this control step)
            if self.nccl_graph:
                self.nccl_graph.replay()
                return
            self.ctx.check(lib.jm_loop_rollout(h, C.c_void_p(self.record.data_ptr())))
            gathered = exchange_records(self.record, self.group)
            self.ctx.check(lib.jm_loop_finish(h, C.c_void_p(gathered.data_ptr()), self.world))
        self._keep = gathered  # alive until the stream consumed it

    def _capture_nccl_step(self):
        """The NCCL transport's step (rollout + reduce, all_gather_into_tensor, finalize) as one CUDA
        graph, replayed per control step: one launch instead of three enqueues and a collective call.
        NCCL collectives are capturable; every rank captures the same sequence.  JM_NCCL_GRAPH=0, or a
        capture that fails on any rank (all ranks then agree to enqueue directly), keeps the direct form."""
        import torch
        import torch.distributed as dist

        lib, h = self.ctx.lib, self.ctx.h
        self.nccl_graph = False
        want = os.environ.get("JM_NCCL_GRAPH", "1") != "0" and self.record.is_cuda
        ok, graph, stepped = want, None, False
        if want:
            dev = self.record.device
            self.gathered = torch.empty((self.world,) + tuple(self.record.shape), dtype=self.record.dtype, device=dev)
            try:
                # one eager step first: NCCL's lazy communicator setup must not happen under capture
                self.ctx.check(lib.jm_loop_rollout(h, C.c_void_p(self.record.data_ptr())))
                dist.all_gather_into_tensor(self.gathered, self.record, group=self.group)
                self.ctx.check(lib.jm_loop_finish(h, C.c_void_p(self.gathered.data_ptr()), self.world))
                torch.cuda.synchronize(dev)
                stepped = True
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=self.stream):
                    self.ctx.check(lib.jm_loop_rollout(h, C.c_void_p(self.record.data_ptr())))
                    dist.all_gather_into_tensor(self.gathered, self.record, group=self.group)
                    self.ctx.check(lib.jm_loop_finish(h, C.c_void_p(self.gathered.data_ptr()), self.world))
            except (RuntimeError, OSError) as exc:
                ok, self.nccl_graph_error = False, exc
        if agree(ok, self.group) and want:
            self.nccl_graph = graph
        return stepped

    def history(self, steps: int):
        """(states (steps+1, n), controls (steps, m), jumps (steps,)) of the loop so far."""
        import torch

        torch.cuda.synchronize(self.ctx.device)
        st = np.empty((steps + 1, self.ctx.N))
        co = np.empty((steps, self.ctx.M))
        ju = np.empty(steps, dtype=np.int64)
        self.ctx.check(self.ctx.lib.jm_loop_history(self.ctx.h, steps, L.dptr(st), L.dptr(co), L.i64ptr(ju)))
        return st, co, ju

    def read(self):
        import torch

        torch.cuda.synchronize(self.ctx.device)  # the steps ran on torch's stream
        lib, h = self.ctx.lib, self.ctx.h
        x = np.zeros(self.ctx.N)
        it, st, hal, status = C.c_uint64(), C.c_int32(), C.c_int32(), C.c_int32()
        self.ctx.check(lib.jm_loop_read(h, L.dptr(x), C.byref(it), C.byref(st), C.byref(hal), C.byref(status)))
        return x, it.value, st.value, hal.value, status.value


def bench_sharded(a, world: int, rank: int, local: int, clock_sampler=None, flops_per_state_step=None):
    """bench.py entry for N > 1 (torchrun): weak scaling (K samples per GPU) or
    strong scaling (BASELINE config 3: K in total, K/N per GPU)."""
    import json
    import time

    import torch
    import torch.distributed as dist

    import paper_1807_06108_b200 as jb

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    idx = {"cfg0": 0, "cfg1": 1, "cfg2": 2, "cfg3": 3}[a.workload]
    task, cfg = jb.baseline_config(idx, K=a.samples, T=a.horizon)
    K, T = cfg.samples_m, cfg.horizon_n
    scaling = getattr(a, "scaling", None) or ("strong" if idx == 3 else "weak")
    n_total = a.warmup + a.steps
    transport = os.environ.get("JM_EXCHANGE", "nccl")
    loop = ShardedLoop.create(task, cfg, rank, world, local, precision=a.precision, transport=transport,
                              scaling=scaling)
    kSettleMax = 20000
    loop.init(task.x0, cfg.u_init, 0, 3 * n_total + 64 + kSettleMax)  # (falls back to NCCL on every rank together)
    k_local = loop.ctx.K
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    t_w = time.perf_counter()
    for _ in range(a.warmup):
        loop.step()
    torch.cuda.synchronize()
    tw = torch.tensor([(time.perf_counter() - t_w) / max(1, a.warmup)], dtype=torch.float64, device="cuda")
    dist.all_reduce(tw, op=dist.ReduceOp.MAX)
    n_settle = int(min(kSettleMax, max(0.0, 1.0 / max(float(tw.item()), 1e-6)))) if clock_sampler is not None else 0
    # the timed steps are enqueued back to back (no host round trip between
    # them, as the device-resident loop runs); per step an L2 flush outside the
    # step's event pair; barrier + synchronize around the whole region
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    import contextlib

    sampler = clock_sampler(local) if (clock_sampler is not None and rank == 0) else contextlib.nullcontext()
    dist.barrier()
    torch.cuda.synchronize()
    with sampler as clk:
        # ~1 s of untimed steps so rank 0's clock record covers a loaded GPU: the same count on
        # every rank (the exchange is collective), from the slowest rank's warm-up pace
        for _ in range(n_settle):
            loop.step()
        torch.cuda.synchronize()
        for i in range(a.steps):
            with torch.cuda.stream(loop.stream):
                flush.fill_(i & 0xFF)  # evict L2 between timed steps
            evs[i][0].record(loop.stream)  # events on the stream the kernels run on
            loop.step()
            evs[i][1].record(loop.stream)
        torch.cuda.synchronize()
    dist.barrier()
    # end to end through the public sharded API: per step the loop's step() and a host read of the
    # plant state it produced (loop.read(): the step's result, device -> host), host wall clock,
    # barrier on both sides, max over ranks; the closed loop has no per-step host input
    h0, d0 = C.c_int64(), C.c_int64()
    h1, d1 = C.c_int64(), C.c_int64()
    loop.ctx.lib.jm_transfer_bytes(C.byref(h0), C.byref(d0))
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        loop.step()
        loop.read()
    e2e_s = (time.perf_counter() - t0) / a.steps
    dist.barrier()
    loop.ctx.lib.jm_transfer_bytes(C.byref(h1), C.byref(d1))
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())
    times = [e0.elapsed_time(e1) for e0, e1 in evs]
    t = torch.tensor([float(np.mean(times))], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max over ranks
    kl = torch.tensor([k_local, -k_local], dtype=torch.int64, device="cuda")
    dist.all_reduce(kl, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    x, it, st, halted, status = loop.read()
    if halted:
        raise RuntimeError(f"sharded loop halted (status {status})")
    if rank == 0:
        value = loop.k_total * T / (ms * 1e-3)
        exch = (("two-level: one reduced record per rank" if loop.two_level else "flat: per-CTA records") +
                " over peer memory (symmetric buffers, device-side epoch flags, no collective launch)"
                if loop.transport == "p2p" else
                "NCCL all_gather_into_tensor of one reduced record per rank")
        line = {"metric": "rollout state-steps/sec (K*T/s)", "value": value, "unit": "state-steps/s",
                "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": a.precision,
                "data": "synthetic",
                "config": {"workload": f"{a.workload}: BASELINE config {idx} closed-loop control step, "
                                       f"K={loop.k_total} in total ({'K/N' if scaling == 'strong' else 'K'} per GPU: "
                                       f"{int(kl[0].item())}{'' if -int(kl[1].item()) == int(kl[0].item()) else ' / ' + str(-int(kl[1].item()))}), "
                                       f"T={T}, one exchange of the weighting records per step",
                           "K_total": loop.k_total, "K_per_gpu_max": int(kl[0].item()), "K_per_gpu_min": -int(kl[1].item()),
                           "exchange": exch, "T": T, "parallelism": f"dp{world}",
                           "l2": "flushed (256 MiB fill) before each timed step"},
                "mpc_iteration_latency_ms": ms, "gpu_launches": loop.launches_per_step() * a.steps}
        line["e2e"] = {"value": loop.k_total * T / e2e_s, "unit": "state-steps/s",
                       "h2d_bytes_per_step": (h1.value - h0.value) // a.steps,
                       "d2h_bytes_per_step": (d1.value - d0.value) // a.steps, "ms_per_step": 1e3 * e2e_s,
                       "path": "ShardedLoop.step() + ShardedLoop.read() (plant state to the host) per control step; "
                               "the closed loop has no per-step host input"}
        if flops_per_state_step is not None:
            # whole-job FP32 rate over the whole step (rollout + exchange + finalize: the rollout kernel is not
            # timed separately here) against N x the live FFMA peak of rank 0's GPU
            peak = engine.microbench(local)["fp32_tflops"] * world
            ach = flops_per_state_step[task.name] * loop.k_total * T / (ms * 1e-3) / 1e12
            line["roofline"] = {"bound": "fp32", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                                "traffic": None, "kernel": loop.ctx.kernel_name() + " (timed: the whole control step)",
                                "flops_per_state_step": flops_per_state_step[task.name]}
        cs = clk.summary() if clk is not None else None
        if cs:
            line["clocks"] = cs
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
