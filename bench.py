#!/usr/bin/env python
"""Benchmark of the B200-native ASA forward (BLADE, arXiv 2508.10774).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl blade|reference]
                    [--workload wan|cog|tiny|wan_stack] [--keep 51 | --tau-mode]

One STEP = one pass of the whole hot path (mask
generation, then block-sparse attention) over one batch of synthetic input.

N = 1 (default): the Wan2.1-1.3B single attention layer of BASELINE.json
    configs[1] (B=1, H=12, N=32760, d=128, bf16, smooth-field inputs,
    keep-ratio 51/256 = sparsity 0.801).  The step is the production single
    call ``blade_asa_fwd``; the same K steps as two calls (``blade_asa_mask``
    + ``blade_bsa_fwd``) give the mask / attention split.  The line also
    carries, as sub-objects, the CogVideoX-5B layer (configs[2]), a sustained
    (~2 s continuous) run of the headline call, and the configs[4] stack on
    one GPU (the N = 1 point of the strong-scaling curve).
N > 1: BASELINE.json configs[4], strong scaling: the Wan2.1-1.3B attention
    stack, batch 8 x 30 layers, 96 (batch, head) units split over the ranks
    (contiguous unit ranges, ``unit_offset`` keys the sampler, inputs seeded
    per GLOBAL unit, so every N computes identical tensors), ``blade_asa_fwd``
    per layer, and the last layer's O gathered to rank 0 over NCCL inside the
    timed step.  ``bench.py --gpus N`` launches its own N ranks (torchrun,
    127.0.0.1) when it is not already running under torchrun.

metric  = BASELINE.json metric: active-block TFLOP/s of the whole ASA call
          (active FLOP = 4 d sum over kept (i,j) valid_i valid_j, probe FLOP
          excluded); value = all ranks' active FLOP / (max over ranks of the
          device time of the K timed steps / K).
e2e     = the same metric through the C ABI with host buffers: pinned host
          Q/K/V -> device, ASA forward, O + LSE -> pinned host, every step.
roofline = attention kernel (the dominant kernel) against the measured bf16
          peak in MEASURED_PEAKS.json.
cpu_baseline = the fp64 oracle (oracle/) on a bounded sample, rank 0, N=1.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2508_10774_b200 import inputs  # noqa: E402

METRIC = "ASA fwd ms/call and effective TFLOPS (active blocks) vs bf16 peak at 1/2/4/8 GPU"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="blade", choices=["blade", "reference"])
    ap.add_argument("--workload", default=None, choices=["wan", "cog", "tiny", "wan_stack"],
                    help="default: wan at N=1, wan_stack at N>1")
    ap.add_argument("--layers", type=int, default=30, help="wan_stack: attention layers per step")
    ap.add_argument("--keep", type=int, default=None,
                    help="keep-ratio mode: lo = hi = KEEP blocks per row (default 51 wan / 25 cog)")
    ap.add_argument("--tau-mode", action="store_true", help="pure tau mode (lo=ceil(.05 Nb), hi=Nb)")
    ap.add_argument("--tau", type=float, default=0.9)
    ap.add_argument("--attn", default="auto", choices=["auto", "tcgen05", "mma", "pair", "triple"])
    ap.add_argument("--variant", default="asa", choices=["asa", "asa_gt"],
                    help="asa_gt: ASA with global tokens (P:135), MeanPool window --window")
    ap.add_argument("--window", type=int, default=128)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunk", type=int, default=0,
                    help="units per chunk of the host-buffer pipeline (0 = library default)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="N=1: skip the cog / sustained / stack sub-measurements")
    ap.add_argument("--sustained-s", type=float, default=2.0)
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_under_torchrun(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: start N ranks of this script."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def mask_params(args, workload: str, Nb: int):
    if args.tau_mode:
        return dict(tau=args.tau, keep_min=max(1, -(-5 * Nb // 100)), keep_max=Nb), "tau"
    keep = args.keep if args.keep is not None else {"wan": 51, "cog": 25, "tiny": 2,
                                                    "wan_stack": 51}[workload]
    keep = min(keep, Nb)
    return dict(tau=args.tau, keep_min=keep, keep_max=keep), f"keep{keep}"


def active_flop(kv_idx: np.ndarray, kv_cnt: np.ndarray, N: int, d: int, b: int = 128) -> float:
    """4 d sum_{u, kept (i, j)} valid_i valid_j."""
    Nb = kv_cnt.shape[1]
    valid = np.array([min(b, N - i * b) for i in range(Nb)], dtype=np.float64)
    live = np.arange(Nb)[None, None, :] < kv_cnt[:, :, None]
    cols = np.where(live, valid[np.clip(kv_idx, 0, Nb - 1)], 0.0).sum(-1)   # [BH, Nb]
    return 4.0 * d * float((cols * valid[None, :]).sum())


def probe_flop(BH, N, d, k=16, b=128):
    Nb = (N + b - 1) // b
    nk = sum(min(k, min(b, N - i * b)) for i in range(Nb))
    return 2.0 * BH * nk * nk * d


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.p = None
        t0 = time.time()  # wait for the first sample so the timed region is covered
        while self.p is not None and time.time() - t0 < 3.0:
            self.f.flush()
            if os.path.getsize(self.f.name) > 0:
                break
            time.sleep(0.02)

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(", ") for r in self.f.read().strip().splitlines() if r.count(",") >= 7]
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "power_w_max": max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit()),
                "samples": len(rows), "reasons": reasons}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except (OSError, ValueError):
        return {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}, "fallback"


def traffic_for(workload: str, kernel: str):
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return t.get(workload, {}).get(kernel)
    except (OSError, ValueError):
        return None


def cores_used() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# CPU oracle legs (the only place bench.py touches oracle/)
# ---------------------------------------------------------------------------


def oracle_sample(q, k, v, N, d, mp, units, qblocks: int | None):
    """Time the fp64 oracle (as it stands) on the first ``units`` units: their
    full mask and the attention of ``qblocks`` evenly spaced query blocks
    per unit (all if None).  Returns (active FLOP of the attention actually
    run, seconds it took, description, mask seconds, attention seconds per
    query block) — no extrapolation."""
    from oracle import asa_oracle as O
    p = O.AsaParams(tau=mp["tau"], keep_min=mp["keep_min"], keep_max=mp["keep_max"])
    t0 = time.perf_counter()
    r = O.asa_mask(q[:units], k[:units], p)
    t_mask = time.perf_counter() - t0
    Nb = r.kv_cnt.shape[1]
    blocks = (list(range(Nb)) if qblocks is None or qblocks >= Nb else
              sorted(set(np.linspace(0, Nb - 1, qblocks).astype(int).tolist())))
    t0 = time.perf_counter()
    O.sparse_attention(q[:units], k[:units], v[:units], r.kv_idx, r.kv_cnt, 128, qblocks=blocks)
    t_att = time.perf_counter() - t0
    valid = np.array([min(128, N - i * 128) for i in range(Nb)], dtype=np.float64)
    flop = sum(4.0 * d * valid[i] * valid[r.kv_idx[u, i, :r.kv_cnt[u, i]]].sum()
               for u in range(units) for i in blocks)
    desc = (f"{units} unit(s) of the layer, fp64 numpy oracle: full mask ({t_mask:.2f} s) + "
            f"attention of {len(blocks)} of {Nb} query blocks per unit ({t_att:.2f} s); value = "
            "active FLOP of the attention actually run / (mask + attention seconds)")
    return flop, t_mask + t_att, desc, t_mask, t_att / (units * len(blocks))


def run_reference(args, ws, rank):
    """--impl reference: the oracle as it stands (there is no reference
    implementation: the reference is a paper), on bounded samples of the same
    workload and metric.  Each of the W + K steps runs the same sample: one
    unit's full mask plus the attention of as many of its query blocks as fit
    a per-step budget that keeps the whole run within ~2-3 minutes; the
    reported time per step is the time of the work actually run."""
    if rank != 0:
        return
    name = args.workload or ("wan" if ws == 1 else "wan_stack")
    w = inputs.WORKLOADS["wan" if name == "wan_stack" else name]
    q, k, v = inputs.smooth(1, 1, w.N, w.d, w.grid, w.n_text, w.ell, w.beta, w.sigma_n, seed=42)
    Nb = (w.N + 127) // 128
    mp, mode = mask_params(args, name, Nb)
    budget_s = float(os.environ.get("BLADE_REF_BUDGET_S", "150"))
    per_step = budget_s / max(1, args.steps + args.warmup)
    # calibrate on a 4-block sample, then size the per-step sample to the budget
    _, _, _, t_mask, t_blk = oracle_sample(q, k, v, w.N, w.d, mp, 1, 4)
    qb = int(max(1, min(Nb, (per_step - t_mask) / max(t_blk, 1e-4))))
    for _ in range(args.warmup):
        oracle_sample(q, k, v, w.N, w.d, mp, 1, qb)
    vals, secs = [], []
    desc = ""
    for _ in range(args.steps):
        flop, sec, desc, _, _ = oracle_sample(q, k, v, w.N, w.d, mp, 1, qb)
        vals.append(flop / sec / 1e12)
        secs.append(sec)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(secs) * 1e3, "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": w.name if name != "wan_stack" else inputs.WORKLOADS[name].name,
                   "B": 1, "H": w.H, "N": w.N, "d": w.d, "mask": mode, "tau": mp["tau"],
                   "sample_per_step": desc, "query_blocks_per_step": qb},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores_used(),
                         "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# CUDA path
# ---------------------------------------------------------------------------


# BLADE_BENCH_SHARE_GPU=1 (testing only): every rank uses cuda:0 and gloo, so
# the multi-rank code path (sharding, max-over-ranks timing, gather) can be
# exercised on a single-GPU box; numbers measured that way are not bench values.
_SHARE_GPU = os.environ.get("BLADE_BENCH_SHARE_GPU") == "1"


def bind_device(local: int) -> torch.device:
    idx = 0 if _SHARE_GPU else local
    torch.cuda.set_device(idx)
    return torch.device("cuda", idx)


def init_dist(dev: torch.device) -> None:
    import torch.distributed as dist
    if _SHARE_GPU:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)


def _ev():
    return torch.cuda.Event(enable_timing=True)


def gpu_head_start(stream) -> None:
    """Keep the GPU busy (~200 ms spin, untimed) while the host enqueues the
    timed calls, so a host-side stall (Python GC, an allocator call, the clock
    sampler) cannot open an idle gap inside the timed region: a 10 ms spin
    still let one 56 ms host stall into a two-call step on the B200."""
    with torch.cuda.stream(stream):
        torch.cuda._sleep(400_000_000)


def time_loop(fn, steps: int, stream) -> float:
    """Mean ms per call of ``steps`` back-to-back calls (CUDA events on the
    launching stream)."""
    e0, e1 = _ev(), _ev()
    gpu_head_start(stream)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def stack_layers(w, args, lo: int, hi: int, dev):
    """Per-layer inputs of the configs[4] stack for GLOBAL units [lo, hi)
    (seed 42 + layer, one generator per global unit: identical at every N)."""
    return [inputs.smooth_device(range(lo, hi), w.N, w.d, w.grid, dev, ell=w.ell, beta=w.beta,
                                 sigma_n=w.sigma_n, seed=42 + layer)
            for layer in range(args.layers)]


def run_stack(args, ws, rank, local, dev, *, sub: bool = False):
    """BASELINE.json configs[4]: the Wan2.1-1.3B attention stack, batch 8 x
    30 layers, (batch, head) units sharded over the ranks (strong scaling:
    the total work is fixed), one ``blade_asa_fwd`` per layer, the last
    layer's O gathered to rank 0 inside the timed step (NCCL)."""
    from paper_2508_10774_b200 import asa as A
    from paper_2508_10774_b200 import shard
    w = inputs.WORKLOADS["wan_stack"]
    units = w.B * w.H
    lo, hi = shard.unit_range(ws, rank, units)
    Nb = (w.N + 127) // 128
    mp, mode = mask_params(args, "wan_stack", Nb)
    layers = stack_layers(w, args, lo, hi, dev)
    stream = torch.cuda.current_stream()
    outs = [None]

    def layer_call(li, q, k, v):
        outs[0] = A.blade_asa_fwd(q, k, v, unit_offset=lo, seed=42 + li, out=outs[0], **mp)
        return outs[0]

    ev_g = [None]

    def step():
        for li, (q, k, v) in enumerate(layers):
            layer_call(li, q, k, v)
        if ev_g[0] is not None:
            ev_g[0].record(stream)
        if ws > 1:
            return shard.gather_units(outs[0][0], units)
        return outs[0][0]

    flop = 0.0
    for li, (q, k, v) in enumerate(layers):  # active FLOP of this rank's units, every layer
        _, _, idx, cnt = layer_call(li, q, k, v)
        flop += active_flop(idx.cpu().numpy(), cnt.cpu().numpy(), w.N, w.d)
    for _ in range(max(args.warmup, 3)):
        step()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk = None if sub else ClockSampler(local)
    e0, e1 = _ev(), _ev()
    gstarts = [_ev() for _ in range(args.steps)]
    gends = [_ev() for _ in range(args.steps)]
    gpu_head_start(stream)
    e0.record(stream)
    for s in range(args.steps):
        ev_g[0] = gstarts[s]
        step()
        gends[s].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop() if clk else None
    ms_local = e0.elapsed_time(e1) / args.steps
    gather_ms_local = statistics.mean(gstarts[s].elapsed_time(gends[s]) for s in range(args.steps))
    ms, gather_ms = shard.max_over_ranks([ms_local, gather_ms_local], device=dev)
    flop_all = shard.sum_over_ranks([flop], device=dev)[0]
    flop_max = shard.max_over_ranks([flop], device=dev)[0]
    ms_min = -shard.max_over_ranks([-ms_local], device=dev)[0]
    o_bytes_to_rank0 = (units - (shard.unit_range(ws, 0, units)[1])) * w.N * w.d * 2
    res = {
        "value": flop_all / (ms * 1e-3) / 1e12, "ms_per_step": ms,
        "ms_per_layer": ms / args.layers, "gather_ms": gather_ms if ws > 1 else 0.0,
        "gather_bytes_to_rank0": o_bytes_to_rank0 if ws > 1 else 0,
        "gather_gbs": (o_bytes_to_rank0 / (gather_ms * 1e-3) / 1e9) if ws > 1 and gather_ms > 0
        else None,
        "rank_imbalance_active_flop": flop_max / (flop_all / ws),
        "rank_time_spread": ms / ms_min if ms_min > 0 else None,
        "units_per_rank": hi - lo, "layers": args.layers, "mask": mode,
        "active_tflop_per_step": flop_all / 1e12,
    }
    if sub or rank != 0:
        return res
    line = {
        "metric": METRIC, "value": res["value"], "unit": "TFLOP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (smooth-field Q/K drawn on device per global unit, iid V; "
                "DESIGN.md §Inputs)",
        "config": {"workload": w.name, "B": w.B, "H": w.H, "N": w.N, "d": w.d,
                   "layers": args.layers, "mask": mode, "units_per_rank": hi - lo,
                   "parallelism": f"(batch,head)-sharded x{ws}; NCCL gather of the last "
                   "layer's O to rank 0 inside the step",
                   "backend": "gloo (shared GPU, testing)" if _SHARE_GPU else "nccl",
                   "l2": "inputs larger than L2, no flush"},
        "ms_per_layer": res["ms_per_layer"], "gather_ms": res["gather_ms"],
        "gather_bytes_to_rank0": res["gather_bytes_to_rank0"], "gather_gbs": res["gather_gbs"],
        "rank_imbalance_active_flop": res["rank_imbalance_active_flop"],
        "rank_time_spread": res["rank_time_spread"], "clocks": clocks,
        "e2e": None,
        "gpu_launches": (5 + int(mp["keep_min"] < mp["keep_max"])) * args.layers * args.steps,
    }
    print(json.dumps(line), flush=True)
    return res


def measure_layer(args, workload: str, dev, local: int, *, headline: bool):
    """One attention layer (BJ configs[1] / configs[2]) on one GPU."""
    from paper_2508_10774_b200 import asa as A

    w = inputs.WORKLOADS[workload]
    q_h, k_h, v_h = inputs.smooth(1, w.H, w.N, w.d, w.grid, w.n_text, w.ell, w.beta, w.sigma_n,
                                  seed=42)
    BH, N, d = q_h.shape
    Nb = (N + 127) // 128
    mp, mode = mask_params(args, workload, Nb)
    impl = {"auto": A.ATTN_AUTO, "tcgen05": A.ATTN_TCGEN05, "mma": A.ATTN_MMA_SYNC,
            "pair": A.ATTN_TCGEN05_PAIR, "triple": A.ATTN_TCGEN05_TRIPLE}[args.attn]
    q, k, v = (t.to(dev) for t in (q_h, k_h, v_h))
    stream = torch.cuda.current_stream()
    gt = args.variant == "asa_gt" and headline
    ev_mid = [_ev()]

    def step():
        if gt:  # ASA_GT: MeanPool_n counts as mask-side work
            kg, vg = A.blade_gt_pool(k, v, window=args.window)
        m = A.blade_asa_mask(q, k, want_mask=False, **mp)
        ev_mid[0].record(stream)
        if gt:
            A.blade_bsa_gt_fwd(q, k, v, m.kv_idx, m.kv_cnt, kg, vg, window=args.window,
                               impl=impl)
        else:
            A.blade_bsa_fwd(q, k, v, m.kv_idx, m.kv_cnt, impl=impl)
        return m

    for _ in range(max(args.warmup, 3)):
        m = step()
    torch.cuda.synchronize()
    kv_idx_np, kv_cnt_np = m.kv_idx.cpu().numpy(), m.kv_cnt.cpu().numpy()
    flop = active_flop(kv_idx_np, kv_cnt_np, N, d)
    if gt:  # every query row also attends the N_g global tokens
        flop += 4.0 * d * BH * N * A.num_global_tokens(N, args.window)
    refined = int(m.n_refined.item())
    sparsity = 1.0 - kv_cnt_np.sum() / (BH * Nb * Nb)

    fo = [None]

    def fused():
        if gt:
            fo[0] = A.blade_asa_gt_fwd(q, k, v, window=args.window, impl=impl, out=fo[0], **mp)
        else:
            fo[0] = A.blade_asa_fwd(q, k, v, impl=impl, out=fo[0], **mp)

    for _ in range(3):
        fused()
    torch.cuda.synchronize()
    clk = ClockSampler(local) if headline else None
    time.sleep(0.3 if headline else 0.0)
    # (1) the production single call: the headline
    fused_ms = time_loop(fused, args.steps, stream)
    # (2) the same K steps as two calls, with an event between them
    starts = [_ev() for _ in range(args.steps)]
    mids = [_ev() for _ in range(args.steps)]
    ends = [_ev() for _ in range(args.steps)]
    gpu_head_start(stream)
    for s in range(args.steps):
        starts[s].record(stream)
        ev_mid[0] = mids[s]
        step()
        ends[s].record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop() if clk else None
    two_ms = statistics.mean(starts[s].elapsed_time(ends[s]) for s in range(args.steps))
    attn_all = [mids[s].elapsed_time(ends[s]) for s in range(args.steps)]
    attn_ms = statistics.mean(attn_all)
    mask_ms = statistics.mean(starts[s].elapsed_time(mids[s]) for s in range(args.steps))
    pk, pk_src = peaks()
    attn_tflops = flop / (attn_ms * 1e-3) / 1e12
    res = {"workload": w.name, "value": flop / (fused_ms * 1e-3) / 1e12,
           "ms_per_step": fused_ms, "ms_mask": mask_ms, "ms_attn": attn_ms,
           "ms_per_step_two_calls": two_ms, "sparsity": round(float(sparsity), 4),
           "rows_refined_fp64": refined, "mask": mode, "keep": [mp["keep_min"], mp["keep_max"]],
           "attn_tflops": attn_tflops, "attn_frac": attn_tflops / pk["bf16_tflops"],
           "active_tflop": flop / 1e12, "steps": args.steps,
           "ms_attn_min_median_max": [min(attn_all), statistics.median(attn_all), max(attn_all)]}
    if not headline:
        return res
    # e2e: host buffers through the ABI, copies inside the timed region
    e2e = None
    if not args.no_e2e and not gt:  # the host-buffer entry point runs plain ASA
        qp, kp, vp = (t.pin_memory() for t in (q_h, k_h, v_h))
        o_host = torch.empty_like(q_h).pin_memory()
        lse_host = torch.empty((BH, N), dtype=torch.float32).pin_memory()

        def e2e_step():
            # the public host-buffer entry point: chunked H2D / compute / D2H overlap
            A.blade_asa_fwd_host(qp, kp, vp, impl=impl, chunk_units=args.e2e_chunk, o=o_host,
                                 lse=lse_host, **mp)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        e2e_ms = time_loop(e2e_step, args.steps, stream)
        e2e = {"value": flop / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": e2e_ms, "api": "blade_asa_fwd_host (C ABI, pinned host buffers, "
               "chunked copy/compute overlap)", "h2d_bytes_per_step": 3 * q_h.numel() * 2,
               "d2h_bytes_per_step": q_h.numel() * 2 + BH * N * 4}
    roof = {"kernel": "attn_tc2p_kernel (persistent pair kernel, blade_bsa_fwd AUTO)",
            "bound": "tensor",
            "achieved": attn_tflops, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
            "frac": attn_tflops / pk["bf16_tflops"],
            "peak_source": f"{pk_src} bf16 burst (MEASURED_PEAKS.json)",
            "traffic": traffic_for(args.workload or "wan", "attn"),
            "attn_ms": attn_ms, "mask_ms": mask_ms, "attn_share": attn_ms / (attn_ms + mask_ms)}
    # the mask side: the sampled probe is exponential- (MUFU-)
    # and tensor-bound, the gather / list writes HBM-bound; all three rates
    # over the whole blade_asa_mask time (sample, probe, select, refine)
    nk = sum(min(16, min(128, N - i * 128)) for i in range(Nb))
    sm_clk = (clocks.get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)) * 1e6
    mufu_peak = 16.0 * 148 * sm_clk  # ex2 per second (16 per clock per SM)
    exps = BH * nk * nk / (mask_ms * 1e-3)
    mask_bytes = BH * (2 * nk * d * 2 + Nb * Nb * 4 + Nb * 4)
    mask_roof = {"bound": "mufu", "basis": "whole blade_asa_mask time",
                 "exps_per_s": exps, "mufu_peak_exps_per_s": mufu_peak,
                 "mufu_frac": exps / mufu_peak,
                 "probe_tflops": probe_flop(BH, N, d) / (mask_ms * 1e-3) / 1e12,
                 "probe_tensor_frac": probe_flop(BH, N, d) / (mask_ms * 1e-3) / 1e12
                 / pk["bf16_tflops"],
                 "hbm_gbs_algorithmic": mask_bytes / (mask_ms * 1e-3) / 1e9,
                 "hbm_frac": mask_bytes / (mask_ms * 1e-3) / 1e9 / pk["hbm_gbs"]}
    res.update(e2e=e2e, roofline=roof, mask_roofline=mask_roof, clocks=clocks,
               flop=flop, BH=BH, N=N, d=d, mp=mp, q_h=q_h, k_h=k_h, v_h=v_h, gt=gt,
               sustained=None)
    # sustained: the headline call back to back for ~args.sustained_s seconds
    if not args.no_extra and args.sustained_s > 0:
        n = max(args.steps, int(args.sustained_s / (fused_ms * 1e-3)))
        clk2 = ClockSampler(local)
        s_ms = time_loop(fused, n, stream)
        res["sustained"] = {"steps": n, "ms_per_step": s_ms,
                            "value": flop / (s_ms * 1e-3) / 1e12, "clocks": clk2.stop(),
                            "peak_for_context": pk.get("bf16_tflops_sustained")}
    return res


def run_single(args, dev, local):
    from paper_2508_10774_b200 import asa as A  # noqa: F401 (fails loudly without the .so)
    workload = args.workload or "wan"
    r = measure_layer(args, workload, dev, local, headline=True)
    extra = {}
    if not args.no_extra and workload == "wan" and not args.tau_mode and args.keep is None:
        extra["cog"] = measure_layer(args, "cog", dev, local, headline=False)
        torch.cuda.empty_cache()
        sub_args = argparse.Namespace(**{**vars(args), "steps": min(args.steps, 10),
                                         "warmup": 3})
        extra["stack_1gpu"] = run_stack(sub_args, 1, 0, local, dev, sub=True)
        torch.cuda.empty_cache()
    cpu = None
    if not args.no_cpu:
        f1, sec, desc, _, _ = oracle_sample(r["q_h"], r["k_h"], r["v_h"], r["N"], r["d"],
                                            r["mp"], 2, None)
        cpu = {"value": f1 / sec / 1e12, "unit": "TFLOP/s", "cores": cores_used(),
               "kind": "oracle", "sample": desc}
    gt = r["gt"]
    mp = r["mp"]
    line = {
        "metric": METRIC, "value": r["value"], "unit": "TFLOP/s", "n_gpus": 1,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": r["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (smooth-field Q/K, iid V; DESIGN.md §Inputs)",
        "config": {"workload": r["workload"], "B": 1, "H": r["BH"], "N": r["N"], "d": r["d"],
                   "variant": args.variant + (f" (window {args.window})" if gt else ""),
                   "mask": r["mask"], "tau": mp["tau"], "keep": r["keep"],
                   "block": 128, "samples": 16, "sparsity": r["sparsity"],
                   "parallelism": "single GPU (the N>1 lines: configs[4] strong scaling)",
                   "attn_impl": args.attn, "l2": "inputs larger than L2 (Q+K+V "
                   f"{3 * r['q_h'].numel() * 2 / 1e6:.0f} MB per step), no flush",
                   "rows_refined_fp64": r["rows_refined_fp64"],
                   "probe_gflop": probe_flop(r["BH"], r["N"], r["d"]) / 1e9},
        "ms_mask": r["ms_mask"], "ms_attn": r["ms_attn"],
        "ms_attn_min_median_max": r["ms_attn_min_median_max"],
        "ms_per_step_two_calls": r["ms_per_step_two_calls"],
        "step_api": ("blade_asa_gt_fwd" if gt else "blade_asa_fwd") +
                    " (one call; attention a programmatic dependent of the mask's last kernel)",
        "clocks": r["clocks"], "e2e": r["e2e"], "roofline": r["roofline"],
        "mask_roofline": r["mask_roofline"], "cpu_baseline": cpu,
        "sustained": r["sustained"],
        "gpu_launches": (5 + int(gt) + int(mp["keep_min"] < mp["keep_max"])) * args.steps,
    }
    for key, val in extra.items():
        line[key] = val
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    in_torchrun = "WORLD_SIZE" in os.environ
    if args.gpus > 1 and not in_torchrun:
        sys.exit(relaunch_under_torchrun(args.gpus))
    ws, rank, local = dist_env()
    if in_torchrun and ws != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}\n")
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    dev = bind_device(local)
    if ws > 1:
        init_dist(dev)
    try:
        if ws > 1 or args.workload == "wan_stack":
            run_stack(args, ws, rank, local, dev)
        else:
            run_single(args, dev, local)
    finally:
        if ws > 1:
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
