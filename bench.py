#!/usr/bin/env python
"""Benchmark of the DS2 CTC loss + gradient hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload english]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...
    python bench.py --impl reference ...     # the reference CPU CTC arm

A "step" is one pass of the CTC hot path over one global minibatch that is
already resident in HBM: ds2ctc_compute_loss (logit stats -> alpha||beta
pair chain with the fused gradient [-> dense gradient]) + the trainer's
{sum loss, #skipped} reduction (ds2ctc_loss_sum) + for N > 1 one NCCL
all-reduce of those two fp64 scalars (trainer.cpp:174-180). Each GPU owns
its LPT shard of the global minibatch (H1 scheduler).

Timing: W untimed warm-up steps (plus an untimed soak of ~0.5 s so clocks
settle and nvidia-smi sees load), then EXACTLY K steps, each bracketed by
CUDA events on the launching stream, with a 256 MiB memset between steps to
flush L2 (the English inputs are 5 MB and would otherwise stay L2-resident);
barrier + synchronize around the timed region; max over ranks. `e2e` is the
same metric through the host-buffer C-ABI call (pinned host activations in,
gradients + costs out, copies inside the timed region), measured before the
device-timed loop.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1512_02595_b200.synth import make_batch, sortagrad_lengths  # noqa: E402

METRIC = "CTC loss+grad utterances/sec"
UNIT = "utt/s"

WORKLOADS = {
    # BASELINE.json configs[1]: the headline (fits one GPU; weak scaling, 64 utterances per GPU)
    "english": dict(A=29, T=700, L=150, per_gpu=64, scaling="weak",
                    desc="English DS2 shape A=29 T=700 L=150, 64 utterances per GPU"),
    "config1": dict(A=29, T=150, L=40, per_gpu=16, scaling="weak", desc="configs[0] A=29 T=150 L=40 B=16 per GPU"),
    "mandarin": dict(A=6000, T=350, L=60, per_gpu=64, scaling="weak",
                     desc="Mandarin DS2 shape A=6000 T=350 L=60, 64 utterances per GPU"),
    "sortagrad": dict(A=29, total=512, scaling="strong",
                      desc="SortaGrad batch T~U[50,1500] L~U[5,min(300,T/2)] B=512 sharded over N GPUs"),
    "edge1500": dict(A=29, T=1500, L=300, total=1024, scaling="strong",
                     desc="B=1024 at T=1500 L=300 sharded over N GPUs"),
    # the CTC step plus its gradient's consumer, the output
    # FC backward (nn.cpp:874-899) on tcgen05, on the device-resident gradient,
    # and for N > 1 the parameter-gradient all-reduce (trainer.cpp:175) over NCCL
    "english-step": dict(A=29, T=700, L=150, per_gpu=64, fc_hidden=2560, scaling="weak",
                         desc="English DS2 shape + output-FC backward (H=2560, the paper's 2560-unit "
                              "model) on the device-resident CTC gradient, 64 utterances per GPU"),
}


def bench_config(name: str, wl: dict, n_gpus: int) -> dict:
    """The workload description both arms print as `config` (identical dicts, so
    the driver can match the arms); arm-specific details go outside it."""
    il_g, ll_g = global_batch(wl, n_gpus)
    return {"workload": name, "desc": wl["desc"], "alphabet": wl["A"], "global_batch": int(il_g.shape[0]),
            "frames_per_step": int(il_g.sum()), "labels_per_step": int(ll_g.sum()),
            "parallelism": f"dp{n_gpus}", "l2": "flushed between steps (256 MiB memset)"}


def global_batch(wl: dict, n_gpus: int, seed: int = 1234):
    """(input_lengths, label_lengths) of the global minibatch."""
    if "per_gpu" in wl:
        B = wl["per_gpu"] * n_gpus
        return np.full(B, wl["T"], np.int32), np.full(B, wl["L"], np.int32)
    if "T" in wl:
        return np.full(wl["total"], wl["T"], np.int32), np.full(wl["total"], wl["L"], np.int32)
    T, L = sortagrad_lengths(wl["total"], seed=7)
    order = np.argsort(T, kind="stable")  # one SortaGrad (epoch 0) minibatch
    return T[order], L[order]


def shard_inputs(wl, il_g, ll_g, idx, rank, seed=1234):
    """Synthetic logits N(0,1) (reference Rng stream) for this rank's utterances."""
    il = il_g[idx]
    ll = ll_g[idx]
    acts, flat, ll, il = make_batch(wl["A"], il, ll, seed=seed + 7919 * rank)
    return acts, flat, ll, il


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling in the background (B200_PROFILING.md recipe)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.proc = None
        self.t0 = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ",".join(str(g) for g in gpus), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sms, maxs, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm, mx, util = float(parts[1]), float(parts[2]), float(parts[3])
            except ValueError:
                continue
            if util <= 0:
                continue
            sms.append(sm)
            maxs.append(mx)
            for name, flag in zip(names, parts[5:9]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": max(maxs) if maxs else None,
                "reasons": sorted(reasons), "samples": len(sms)}


def cpu_reference_rate(acts, flat, ll, il, nthreads, min_seconds):
    """The reference's own ctc_loss_reference (oracle/_ref build) on host cores; utt/s.
    Also returns the last call's (costs, grads): the reference's answer on these
    inputs, which the parity gate compares with the GPU's."""
    import oracle

    kind = "reference" if oracle.ref_available() else "port"
    fn = oracle.ref_batch if kind == "reference" else oracle.oracle_batch
    fn(acts[:, :min(4, acts.shape[1]), :], flat[:int(ll[:4].sum())], ll[:4], il[:4], nthreads=nthreads)  # warm
    done = 0
    t0 = time.perf_counter()
    while True:
        out = fn(acts, flat, ll, il, nthreads=nthreads)
        done += ll.shape[0]
        el = time.perf_counter() - t0
        if el >= min_seconds:
            break
    return done / el, kind, done, el, out


def parity_gate(costs, grads, ref_costs, ref_grads, il):
    """SURVEY.md §8(d) same-run parity gate: per utterance |cost - ref| / |ref| <= 1e-4,
    max |grad - ref| <= 1e-4; infeasible -> +inf and all-zero rows (NaN patterns must match)."""
    costs = np.asarray(costs, np.float64)
    ref_costs = np.asarray(ref_costs, np.float64)
    inf_ok = bool(np.array_equal(np.isposinf(costs), np.isposinf(ref_costs)))
    nan_ok = bool(np.array_equal(np.isnan(costs), np.isnan(ref_costs)))
    fin = np.isfinite(ref_costs)
    rel = float((np.abs(costs[fin] - ref_costs[fin]) / np.maximum(np.abs(ref_costs[fin]), 1e-30)).max()) \
        if fin.any() else 0.0
    g = np.asarray(grads, np.float64)
    r = np.asarray(ref_grads, np.float64)
    gnan_ok = bool(np.array_equal(np.isnan(g), np.isnan(r)))
    gerr = float(np.nanmax(np.abs(g - r))) if g.size else 0.0
    for b in np.where(np.isposinf(ref_costs))[0]:
        inf_ok = inf_ok and bool(np.all(g[:, b, :] == 0))
    ok = inf_ok and nan_ok and gnan_ok and rel <= 1e-4 and gerr <= 1e-4
    return {"utterances": int(costs.shape[0]), "max_rel_cost": rel, "max_abs_grad": gerr,
            "tolerance": {"rel_cost": 1e-4, "abs_grad": 1e-4}, "ok": ok}


def run_reference(args, wl):
    """--impl reference: the reference CPU CTC with all host threads (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle

    il_g, ll_g = global_batch(wl, args.gpus)
    n = min(64, il_g.shape[0])
    acts, flat, ll, il = shard_inputs(wl, il_g, ll_g, np.arange(n), 0)
    nthreads = os.cpu_count() or 1
    kind = "reference" if oracle.ref_available() else "port"
    fn = oracle.ref_batch if kind == "reference" else oracle.oracle_batch
    for _ in range(max(args.warmup, 1)):
        fn(acts, flat, ll, il, nthreads=nthreads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fn(acts, flat, ll, il, nthreads=nthreads)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.mean(times)
    value = n / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.workload, wl, args.gpus),
        "sample": {"utterances_per_step": n, "frames_per_step": int(il.sum()),
                   "note": "each step is a bounded sample of the workload's global batch (the first n utterances)"},
        "frames_per_s": float(il.sum()) / (ms / 1e3),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": kind,
                         "sample": f"{n} utterances of the {args.workload} workload per step, "
                                   f"asr::ctc::ctc_loss_reference fp64, one utterance per thread"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# The contract is ONE JSON line on stdout; native libraries (NCCL's
# "NCCL version" banner at communicator init) print to fd 1 directly, so fd 1
# is pointed at stderr and the JSON line goes to a saved copy of the original.
_JSON_OUT = None


def claim_stdout() -> None:
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w", buffering=1)
    os.dup2(2, 1)


def emit(line: dict) -> None:
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="english", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--soak-seconds", type=float, default=0.5)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, wl)

    import torch
    import torch.distributed as dist

    from paper_1512_02595_b200 import _lib, ctc, scheduler

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.lib()

    il_g, ll_g = global_batch(wl, world)
    idx = scheduler.shard_batch(il_g, ll_g, wl["A"], world, rank)
    acts_h, flat, ll, il = shard_inputs(wl, il_g, ll_g, idx, rank)
    B = int(ll.shape[0])
    A = wl["A"]
    x = torch.from_numpy(acts_h).to(dev)
    grads = torch.empty_like(x)
    costs = torch.empty(max(B, 1), dtype=torch.float32, device=dev)
    pair = torch.zeros(2, dtype=torch.float64, device=dev)
    ws = ctc.Workspace(dev)
    ws_ptr, ws_bytes = ws.get(ctc.workspace_size(ll, il, A))
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    P = ctypes.POINTER(ctypes.c_int)
    lab_c = np.ascontiguousarray(flat if flat.size else np.zeros(1, np.int32), dtype=np.int32)
    ll_c = np.ascontiguousarray(ll if B else np.zeros(1, np.int32), dtype=np.int32)
    il_c = np.ascontiguousarray(il if B else np.zeros(1, np.int32), dtype=np.int32)
    launches_per_step = 0

    # N > 1: the scalar sums and their all-reduce are one kernel over NVLink
    # peer memory (ds2ctc_loss_sum_allreduce); DS2CTC_NCCL_REDUCE=1 uses
    # ds2ctc_loss_sum + an NCCL all-reduce instead (the baseline).
    peer = None
    if world > 1 and os.environ.get("DS2CTC_NCCL_REDUCE") != "1":
        from paper_1512_02595_b200.dist import PeerLossReducer

        peer = PeerLossReducer(dev)
        if not peer.ok:  # e.g. no CUDA IPC between the ranks' GPUs: the NCCL baseline
            if rank == 0:
                print(f"peer all-reduce unavailable ({peer.error}); using NCCL", file=sys.stderr)
            peer = None

    # f1: the output layer's cached input, weight and parameter gradients (random init)
    H = wl.get("fc_hidden", 0)
    if H:
        gen = torch.Generator(device=dev)
        gen.manual_seed(4321 + rank)
        fc_x = torch.randn((x.shape[0], B, H), generator=gen, device=dev, dtype=torch.float32)
        fc_w = torch.randn((A, H), generator=gen, device=dev, dtype=torch.float32) * 0.02
        # dW and db in one buffer: one parameter-gradient all-reduce per step
        fc_grad = torch.zeros(A * H + A, device=dev, dtype=torch.float32)
        fc_dw = fc_grad[:A * H].view(A, H)
        fc_db = fc_grad[A * H:]
        vec = None  # f4 over NVLink peer memory (ds2ctc_vec_allreduce); NCCL when unavailable
        if world > 1 and os.environ.get("DS2CTC_NCCL_REDUCE") != "1":
            from paper_1512_02595_b200.dist import PeerVecReducer

            vec = PeerVecReducer(A * H + A, dev)
            if not vec.ok:
                if rank == 0:
                    print(f"peer vector all-reduce unavailable ({vec.error}); using NCCL", file=sys.stderr)
                vec = None
        fc_dx = torch.empty((x.shape[0], B, H), device=dev, dtype=torch.float32)
        fc_ws = ctc.Workspace(dev)
        fc_sz = ctypes.c_size_t()
        _lib.check(lib.ds2ctc_fc_backward_workspace_size(x.shape[0] * B, A, H, ctypes.byref(fc_sz)), "fc ws")
        fc_ws_ptr, fc_ws_bytes = fc_ws.get(int(fc_sz.value))

    def fc_step():
        fc_dw.zero_()  # zero_grads (trainer.cpp:152)
        fc_db.zero_()
        _lib.check(lib.ds2ctc_fc_backward(ctypes.c_void_p(grads.data_ptr()), ctypes.c_void_p(fc_x.data_ptr()),
                                          ctypes.c_void_p(fc_w.data_ptr()), ctypes.c_void_p(fc_dw.data_ptr()),
                                          ctypes.c_void_p(fc_db.data_ptr()), ctypes.c_void_p(fc_dx.data_ptr()),
                                          x.shape[0] * B, A, H, ctypes.c_void_p(fc_ws_ptr), fc_ws_bytes,
                                          ctypes.c_void_p(stream.cuda_stream)), "ds2ctc_fc_backward")
        if world > 1:  # f4: the parameter-gradient all-reduce (trainer.cpp:175, ring_allreduce)
            if vec is not None:
                vec.reduce(fc_grad.data_ptr(), stream.cuda_stream)
            else:
                dist.all_reduce(fc_grad)

    def step(reduce_mode=None):
        st = lib.ds2ctc_compute_loss_checked(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(grads.data_ptr()),
                                             lab_c.ctypes.data_as(P), ll_c.ctypes.data_as(P),
                                             il_c.ctypes.data_as(P), A, B, A - 1, ctypes.c_void_p(costs.data_ptr()),
                                             ctypes.c_void_p(ws_ptr), ws_bytes, ctypes.c_void_p(stream.cuda_stream))
        _lib.check(st, "ds2ctc_compute_loss")
        if H:
            fc_step()
        if peer is not None and reduce_mode != "nccl":
            peer.reduce(costs.data_ptr(), B, pair.data_ptr(), stream.cuda_stream)
            return
        _lib.check(lib.ds2ctc_loss_sum(ctypes.c_void_p(costs.data_ptr()), B, ctypes.c_void_p(pair.data_ptr()),
                                       ctypes.c_void_p(stream.cuda_stream)), "ds2ctc_loss_sum")
        if world > 1:
            dist.all_reduce(pair)

    if H and world > 1 and vec is not None:  # the peer-memory vector all-reduce must agree with NCCL's
        gen_chk = torch.Generator(device=dev)
        gen_chk.manual_seed(99 + rank)
        probe = torch.randn(A * H + A, generator=gen_chk, device=dev, dtype=torch.float32)
        ref_v = probe.clone()
        dist.all_reduce(ref_v)
        fc_grad.copy_(probe)
        vec.reduce(fc_grad.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        vec.check()
        if not torch.allclose(fc_grad, ref_v, rtol=1e-5, atol=1e-5):
            raise RuntimeError("peer vector all-reduce disagrees with NCCL")
    if peer is not None:  # the fused reduction must agree with NCCL's
        step("nccl")
        ref_pair = pair.clone()
        step()
        torch.cuda.synchronize()
        if not torch.allclose(pair, ref_pair, rtol=1e-12, atol=0):
            raise RuntimeError(f"peer all-reduce {pair.tolist()} != NCCL {ref_pair.tolist()}")

    dense_overlap = os.environ.get("DS2CTC_DENSE_OVERLAP", "0") != "0"  # the library's default (ctc_api.cpp): off
    # kernels of ours per step: k_pair (+ k_dense + k_finalize for large A) + k_loss_sum / k_loss_allreduce
    if B:
        # large A: k_dense + k_finalize, or (overlapped) k_dense_soft + k_dense_patch + k_finalize
        launches_per_step = (1 + ((3 if dense_overlap else 2) if A > 128 else 0) + 1
                             + (5 if H else 0)  # fc: pad, bias, W^T, 2 GEMMs
                             + (1 if H and world > 1 and vec is not None else 0))  # f4 peer all-reduce
    else:
        launches_per_step = 1

    # ---- e2e through the host-buffer C-ABI (pinned host buffers, copies timed) ----
    # Measured first, before the sustained device-timed loop: run after it, the
    # same synchronous calls took ~520 us instead of ~370 us on the same box
    # (post-load state; tools/e2e_probe.py reproduces ~380 us standalone).
    acts_pin = torch.from_numpy(acts_h).pin_memory()
    grads_pin = torch.empty(acts_h.shape, dtype=torch.float32).pin_memory()
    costs_pin = torch.empty(max(B, 1), dtype=torch.float32).pin_memory()

    def e2e_call():
        if B == 0:
            return
        st = lib.ds2ctc_compute_loss_host(ctypes.c_void_p(acts_pin.data_ptr()), ctypes.c_void_p(grads_pin.data_ptr()),
                                          lab_c.ctypes.data_as(P), ll_c.ctypes.data_as(P), il_c.ctypes.data_as(P),
                                          A, B, A - 1, ctypes.c_void_p(costs_pin.data_ptr()), local_rank)
        _lib.check(st, "ds2ctc_compute_loss_host")

    # at least 10 untimed calls: the first ones size the per-thread device
    # context (cudaMalloc) and fault in the pinned buffers
    for _ in range(max(args.warmup, 10)):
        e2e_call()
    if world > 1:
        dist.barrier()
    e2e_times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        e2e_call()
        e2e_times.append(time.perf_counter() - t0)
    e2e_ms_local = 1e3 * statistics.mean(e2e_times)

    sampler = ClockSampler([local_rank]) if rank == 0 else None
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # Soak: the same NUMBER of steps on every rank (a per-rank wall-clock loop
    # can end one step apart, which leaves the peer mailboxes' sequence
    # numbers one step out of phase: the last step of the rank ahead then
    # waits for a peer step that never comes). Rank-local estimate, max over ranks.
    t_soak = time.perf_counter()
    for _ in range(3):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    per_step = max((time.perf_counter() - t_soak) / 3, 1e-6)
    n_soak = torch.tensor([int(args.soak_seconds / per_step)], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(n_soak, op=dist.ReduceOp.MAX)
    for _ in range(int(n_soak.item())):
        flush.zero_()
        step()
        if _ % 16 == 15:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    if peer is not None:
        peer.check()  # a timed-out peer wait is an error, never a number

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.zero_()
        starts[k].record(stream)
        step()
        ends[k].record(stream)
    torch.cuda.synchronize()
    if peer is not None:
        peer.check()
    if H and vec is not None:
        vec.check()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    # Per-kernel stage times from the library's own events, in a separate pass
    # after the timed region (its extra event records are not in `value`).
    n_prof = min(args.steps, 20)
    stage = np.zeros((max(n_prof, 1), 4), dtype=np.float64)
    ms4 = (ctypes.c_float * 4)()
    lib.ds2ctc_profile_enable(n_prof if B else 0)
    for k in range(n_prof):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    for k in range(n_prof if B else 0):
        _lib.check(lib.ds2ctc_profile_read(k, ms4), "ds2ctc_profile_read")
        stage[k] = list(ms4)
    lib.ds2ctc_profile_enable(0)
    fc_ms_local = 0.0
    if H:  # the FC backward alone (events on the launching stream), L2 flushed before each
        fe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_prof)]
        for k in range(n_prof):
            flush.zero_()
            fe[k][0].record(stream)
            fc_step()
            fe[k][1].record(stream)
        torch.cuda.synchronize()
        fc_ms_local = statistics.mean(a.elapsed_time(b) for a, b in fe)
    ms_local = statistics.mean(step_ms)
    pair_ms_local = float(stage[:, 0].mean()) if B else 0.0
    dense_ms_local = float(stage[:, 1].mean()) if B else 0.0
    final_ms_local = float(stage[:, 2].mean()) if B else 0.0

    # ---- max over ranks ----
    vals = torch.tensor([ms_local, pair_ms_local, e2e_ms_local, dense_ms_local, final_ms_local, fc_ms_local],
                        dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, pair_ms, e2e_ms, dense_ms, final_ms, fc_ms = [float(v) for v in vals.cpu()]
    total_utts = int(il_g.shape[0])
    total_frames = int(il_g.sum())
    value = total_utts / (ms / 1e3)
    # loss check (parity is the test suite's job; this guards the bench itself)
    torch.cuda.synchronize()
    loss_sum, skipped = [float(v) for v in pair.cpu()]

    if rank == 0:
        peak, peak_kind = load_peaks()
        # Algorithmic bytes of the path: activations read once + gradients
        # written once (8*T*A per utterance) + labels and lengths. Attributed to the dominant
        # kernel: k_pair for small alphabets (it reads the logits and writes the gradient),
        # k_dense for large ones (the HBM pass).
        alg_bytes = 8.0 * float((il.astype(np.float64) * A).sum()) + 4.0 * float(ll.sum()) + 8.0 * B
        dense_name = "k_dense_soft (k_dense_t<V, true>)" if dense_overlap else "k_dense (k_dense_t<V, false>)"
        dom_name, dom_ms = ("k_pair", pair_ms) if A <= 128 else (dense_name, dense_ms)
        achieved = alg_bytes / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else 0.0
        # DRAM bytes per launch of the dominant kernel from one `ncu --set full`
        # capture (tools/ncu/traffic.py), valid only for the exact library it was
        # measured on: profiles/ncu_traffic.json is stamped with the content hash
        # of the sources the library was built from (libds2ctc.so.sha256).
        traffic, traffic_src = None, "no capture for this build"
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        try:
            with open(tpath) as f:
                tj = json.load(f)
            with open(_lib.LIB_PATH + ".sha256") as f:
                lib_hash = f.read().strip()
            if tj.get("lib_sha256") == lib_hash and args.workload in tj.get("bytes", {}):
                traffic = float(tj["bytes"][args.workload])
                traffic_src = f"profiles/ncu_traffic.json ({tj.get('kernel', dom_name)}, build {lib_hash[:12]})"
            else:
                traffic_src = "profiles/ncu_traffic.json is from another build (source hash mismatch)"
        except Exception as exc:  # noqa: BLE001
            traffic_src = f"unavailable ({type(exc).__name__})"
        # The binding bound at small alphabets is the serial lattice chain, not HBM
        # (DESIGN.md §5.1): each CTA of k_pair runs T_max dependent steps. Report the
        # measured cycles per step beside the isolated-step floor measured by
        # tools/microbench/chain_step.cu (one chain warp, K label pairs per lane, the
        # product arithmetic, no service/gradient/halo work), per K of the launch
        # (pick_K, ds2ctc_internal.h; K=1 and K=8 use the nearest measured K).
        sm_mhz = (clocks or {}).get("sm_mhz") or 1965.0
        # Serial steps of the launch: each utterance is two CTAs of T_b steps
        # (one per SM); with more CTAs than SMs, the LPT makespan of those
        # chains over the SMs (the launch order is longest first).
        import heapq

        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        loads = [0] * n_sm
        for t_b in sorted((int(v) for v in il for _ in range(2)), reverse=True):
            heapq.heapreplace(loads, loads[0] + t_b)
        t_steps = max(loads) if il.size else 0
        pairs = int(ll_g.max()) + 1 if ll_g.size else 1
        K = next((k for k in (1, 2, 3, 4, 6, 8) if pairs <= 3 * 28 * k), 8)
        floor = {1: 186.0, 2: 186.0, 3: 214.0, 4: 285.0, 6: 368.5, 8: 368.5}[K]
        chain = None
        if t_steps > 0 and pair_ms > 0:
            cps = pair_ms * 1e-3 * sm_mhz * 1e6 / t_steps
            chain = {"bound": "serial lattice chain (dependent steps per SM: T_max, or the LPT makespan "
                              "of 2 chains of T_b steps per utterance over the SMs)", "steps": t_steps,
                     "pairs_per_lane": K, "cycles_per_step": cps, "floor_cycles_per_step": floor,
                     "frac": floor / cps,
                     "floor_source": "tools/microbench/chain_step.cu (profiles/r01_microbench_chain_step.txt)"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": wl["scaling"],
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": bench_config(args.workload, wl, world),
            "scalar_reduce": ("nvlink peer mailboxes (ds2ctc_loss_sum_allreduce)" if peer is not None
                              else ("nccl all_reduce" if world > 1 else "none")),
            "frames_per_s": total_frames / (ms / 1e3),
            "stage_ms": {"k_pair": pair_ms,
                         ((("k_dense_soft (concurrent with k_pair)" if dense_overlap else "k_dense") if A > 128
                           else "dense pass (none: fused into k_pair)")): dense_ms,
                         "k_finalize": final_ms},
            "roofline": {"bound": "hbm", "kernel": dom_name, "kernel_ms": dom_ms, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_source": traffic_src, "alg_bytes_per_launch": alg_bytes,
                         "chain": chain},
            "e2e": {"value": total_utts / (e2e_ms / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": int(acts_h.nbytes + 4 * (ll.sum() + 2 * B)),
                    "d2h_bytes_per_step": int(acts_h.nbytes + 4 * B), "ms_per_step": e2e_ms},
            # north_star (1): the log-softmax over the alphabet (log_softmax_rows, ctc.cpp:24-37).
            # Large alphabets: it is the dense pass itself (row max + log-sum-exp, the softmax
            # row written with the gradient), reported as achieved GB/s. Small ones: fused
            # into k_pair's service warp (the logits are staged once, per epoch, while the
            # chain runs; epoch timing shows it off the critical path: DESIGN.md section 5.1),
            # so it has no launch or GB/s of its own.
            "log_softmax": ({"kernel": dense_name, "ms": dense_ms,
                             "bytes": 8.0 * float((il.astype(np.float64) * A).sum()),
                             "achieved_gbs": 8.0 * float((il.astype(np.float64) * A).sum()) / (dense_ms / 1e3) / 1e9
                             if dense_ms > 0 else 0.0,
                             "frac": (8.0 * float((il.astype(np.float64) * A).sum()) / (dense_ms / 1e3) / 1e9) / peak
                             if dense_ms > 0 else 0.0,
                             "loads": "float4 rows, L1 no-allocate; block max / sum by warp shuffles"}
                            if A > 128 else
                            {"kernel": "fused into k_pair (service warp)", "bytes_read": 4.0 * float(
                                (il.astype(np.float64) * A).sum()),
                             "note": "one coalesced row read per frame, max / log-sum-exp in the same pass; "
                                     "latency-hidden behind the lattice chain, no separate HBM pass"}),
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "loss_sum": loss_sum, "skipped": int(skipped),
        }
        if H:
            # f1: the FC backward is HBM-bound at A = 29 (K = 29 for dx): x read once for
            # dW, dx written once, the gradient read twice, W / W^T / dW negligible
            rows = x.shape[0] * B
            fc_bytes = 4.0 * (2 * rows * H + 2 * rows * A + 3 * A * H)
            fc_flops = 2.0 * 2 * rows * A * H
            line["fc_backward"] = {"ms": fc_ms, "rows": rows, "in_dim": H, "out_dim": A, "alg_bytes": fc_bytes,
                                   "achieved_gbs": fc_bytes / (fc_ms / 1e3) / 1e9 if fc_ms else None,
                                   "frac_hbm": fc_bytes / (fc_ms / 1e3) / 1e9 / peak if fc_ms else None,
                                   "tflops": fc_flops / (fc_ms / 1e3) / 1e12 if fc_ms else None,
                                   "kernels": "tcgen05 kind::tf32 (k_fc_gemm x2) + bias sum + W^T + row pad",
                                   "param_grad_allreduce": ("nvlink peer memory (ds2ctc_vec_allreduce, dW + db)"
                                                            if world > 1 and vec is not None else
                                                            "nccl all_reduce (dW + db)" if world > 1 else "none")}
        if world == 1 and not args.no_cpu_baseline:
            # The reference CPU CTC on the same inputs: (i) all host cores, one
            # utterance per thread (the paper's CPU CTC); (ii) one
            # core, the trainer's serial loop (trainer.cpp:158-169). Its answers
            # on the sample are the same-run parity gate for the GPU's.
            n = min(64, B)
            sub = np.arange(n)
            nl = int(ll[:n].sum())
            t_n = int(il[:n].max()) if n else 0
            rate, kind, done, el, (rc, rg) = cpu_reference_rate(
                np.ascontiguousarray(acts_h[:t_n, sub, :]), flat[:nl], ll[:n], il[:n], os.cpu_count() or 1,
                args.cpu_seconds)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": kind,
                                    "sample": f"{done} utterances ({n} per batch) of the {args.workload} "
                                              f"workload in {el:.1f} s, asr::ctc::ctc_loss_reference fp64, "
                                              f"one utterance per thread"}
            n1 = min(8, n)
            rate1, kind1, done1, el1, _ = cpu_reference_rate(
                np.ascontiguousarray(acts_h[:int(il[:n1].max()), :n1, :]), flat[:int(ll[:n1].sum())], ll[:n1],
                il[:n1], 1, args.cpu_seconds / 2)
            line["cpu_baseline_serial"] = {"value": rate1, "unit": UNIT, "cores": 1, "kind": kind1,
                                           "sample": f"{done1} utterances ({n1} per batch) in {el1:.1f} s, one "
                                                     f"core, serial as train_epoch calls it (trainer.cpp:158-169)"}
            g_host = grads.cpu().numpy()[:t_n, :n, :] if B else np.zeros((0, 0, A), np.float32)
            line["parity"] = parity_gate(costs.cpu().numpy()[:n], g_host, rc, rg, il[:n])
            line["parity"]["checker"] = f"{kind} ({'oracle/_ref build of ctc_loss_reference' if kind == 'reference' else 'oracle port'}), first {n} utterances of the timed batch"
        emit(line)
    if world > 1:
        dist.barrier()
        if peer is not None:
            torch.cuda.synchronize()
            peer.close()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
