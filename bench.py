#!/usr/bin/env python
"""Benchmark of the MORLAX data-parallel training step on B200.

metric: env-steps/s of one full training iteration (sampling + rollout +
GAE/normalise + 4 epochs x 8 minibatches of PPO through the hypernetwork +
Adam), whole job, as BASELINE.json names. Default workload = config 3 shapes
(8192 mo-humanoid6 envs, T=64, 128 preference clusters, policy
45-256-256-12, critic 45-256-256-6, hypernet 6-256-F256) with config 4's PPO
schedule; weak-scaled per GPU under torchrun (--gpus N: N x 8192 envs,
N x 128 clusters).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c3|pr1]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASE = {
    "c3": dict(env_name="mo-humanoid6", N=8192, K=128, kappa=0, T=64, epochs=4, minibatch_count=8,
               gamma=0.99, gae_lambda=0.95, clip_eps=0.2, actor_lr=3e-4, critic_lr=1e-3,
               entropy_coef=0.01, seed=2, F=256, feature_hidden=[256], actor_hidden=[256, 256],
               critic_hidden=[256, 256]),
    "pr1": dict(env_name="mo-pointmass", N=256, K=16, kappa=0, T=32, epochs=4, minibatch_count=4,
                gamma=0.99, gae_lambda=0.95, clip_eps=0.2, actor_lr=3e-4, critic_lr=3e-4,
                entropy_coef=0.1, seed=0, F=64, feature_hidden=[64], actor_hidden=[64, 64],
                critic_hidden=[64, 64]),
}
WORKLOAD = {"c3": "config3-humanoid6-8192env-T64-128pref (+config4 PPO 4x8)",
            "pr1": "PR1-pointmass-256env-T32-16pref"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops_sustained"], "measured"
    return 6650.0, 1400.0, "fallback"


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(self.idx), "-lms", "200"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.out = ""

    def summary(self):
        sm, mx, reasons = [], None, set()
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"), f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- CPU baseline
def reference_sample(base, cores):
    """Bounded sample of the REFERENCE CPU path (compiled /root/reference
    sources, oracle/_ref) on this host: one iteration of the train() loop
    body on a reduced cluster count K_s (same per-cluster env count, T, row
    count per cluster per minibatch, parameter counts), with one minibatch of
    actor+critic loss and Adam; extrapolated linearly to the full iteration:
      t = (rollout+gae) K/K_s + epochs*mbs*(loss K/K_s + adam)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle, RefTrainer, TrainCfg
    r = Oracle("ref")
    reps = base["N"] // base["K"]
    Ks = base["K"] if base["K"] * reps <= 512 else 2
    cfg = TrainCfg(env=base["env_name"], N=Ks * reps, K=Ks, kappa=base["kappa"], T=base["T"],
                   epochs=base["epochs"], minibatch_count=base["minibatch_count"], gamma=base["gamma"],
                   lam=base["gae_lambda"], clip_eps=base["clip_eps"], actor_lr=base["actor_lr"],
                   critic_lr=base["critic_lr"], entropy_coef=base["entropy_coef"], seed=base["seed"],
                   F=base["F"], feat_hidden=base["feature_hidden"], actor_hidden=base["actor_hidden"],
                   critic_hidden=base["critic_hidden"])
    t = RefTrainer(r, cfg, threads=cores)
    full_mb = Ks == base["K"]
    secs, _, _ = t.iteration(0, -1 if full_mb else 1)
    roll, gae, upd, done, loss_s, adam_s = secs
    scale = base["K"] / Ks
    n_mb = base["epochs"] * base["minibatch_count"]
    if full_mb:
        t_iter = roll + gae + upd
        sample = f"1 full reference iteration ({base['N']} envs)"
    else:
        t_iter = (roll + gae) * scale + n_mb * (loss_s * scale + adam_s)
        sample = (f"reference train() loop body on {Ks} of {base['K']} clusters ({Ks * reps} envs x T={base['T']}),"
                  f" 1 of {n_mb} minibatches (loss {loss_s:.2f}s, adam {adam_s:.2f}s), rollout {roll:.2f}s;"
                  f" extrapolated x{scale:.0f} clusters, x{n_mb} minibatches")
    value = base["N"] * base["T"] / t_iter
    return value, sample, float(roll + gae + upd)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    base = dict(BASE[args.config])
    base["N"] *= world
    base["K"] *= world
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    vals = []
    sample = ""
    for i in range(args.warmup + args.steps):
        v, sample, _ = reference_sample(BASE[args.config] if world == 1 else base, cores)
        if i >= args.warmup:
            vals.append(v)
    v = float(np.median(vals))
    print(json.dumps({
        "impl": "reference", "metric": "env-steps/s", "value": v, "unit": "env-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD[args.config], "envs": base["N"], "clusters": base["K"],
                   "T": base["T"], "parallelism": f"cpu-threads{cores}"},
        "cpu_baseline": {"value": v, "unit": "env-steps/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": v, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ---------------------------------------------------------------- other BASELINE configs (rank 0, N = 1)
def _events_ms(stream, fn, iters):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(iters):
        fn(i)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def leg_pr1(mb, cpu):
    """Config 1 (PR1): mo-pointmass, 256 envs x T 32, 16 preferences, full
    training iteration; the reference's full iteration beside it."""
    import torch
    cfg = mb.TrainConfig(**BASE["pr1"])
    t = mb.Trainer(cfg)
    stream = torch.cuda.ExternalStream(mb.LIB.morlax_trainer_stream(t._h))
    for i in range(3):
        t.iteration(i)
    ms = _events_ms(stream, lambda i: t.iteration(3 + i), 10)
    out = {"workload": WORKLOAD["pr1"], "metric": "env-steps/s", "value": cfg.N * cfg.T / (ms / 1e3),
           "ms_per_step": ms}
    if cpu:
        v, sample, _ = reference_sample(BASE["pr1"], os.cpu_count() or 1)
        out["cpu_reference"] = {"value": v, "unit": "env-steps/s", "cores": os.cpu_count(), "sample": sample}
    return out


def leg_c2(mb, tflops_peak):
    """Config 2: hypernetwork + per-preference policy forward microbench: 64
    preferences ~ Dirichlet(1,1,1), 2048 N(0,1) observations each (131072
    rows, obs 48, act 12); hypernet 3 -> 256 -> F 256, policy 48-256-256-12,
    bf16 operands / fp32 accumulation; reference init (seeded) in place of
    Xavier."""
    import torch
    G, R = 64, 2048
    spec = mb.HypernetSpec(3, 256, [256], [48, 256, 256, 12], True, True)
    pf = mb.PolicyForward(spec, G, R)
    pf.set_params(mb.init_hypernet(spec, mb.rng_words(1, 0, 1)[0]))
    rng = np.random.default_rng(1)
    w = torch.tensor(rng.dirichlet(np.ones(3), size=G), dtype=torch.float32, device="cuda")
    obs = torch.tensor(rng.normal(size=(G * R, 48)), dtype=torch.float32, device="cuda")
    pre = torch.empty((G * R, 12), dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    fwd = lambda i: pf.forward_device(w.data_ptr(), obs.data_ptr(), pre.data_ptr(), stream.cuda_stream)
    for i in range(3):
        fwd(i)
    ms = _events_ms(stream, fwd, 20)
    tf = pf.flops / (ms / 1e3) / 1e12
    return {"workload": "config2-hypernet+policy-forward-64pref-x2048obs", "metric": "forward_us",
            "value": ms * 1e3, "unit": "us", "rows_per_s": G * R / (ms / 1e3), "gflop": pf.flops / 1e9,
            "tflops": tf, "roofline": {"bound": "tensor", "achieved": tf, "peak": tflops_peak,
                                       "unit": "TFLOP/s", "frac": tf / tflops_peak}}


def leg_c4(mb):
    """Config 4: GAE + PPO update on 262144 synthetic transitions (4096 envs x
    T 64): rewards / values ~ N(0,1) (6 objectives), next_value = the next
    step's value (one extra draw at T-1), terminated ~ Bernoulli(0.01),
    64 preference groups ~ Dirichlet(1^6), obs ~ N(0,1), actions ~ N(0,1),
    old log-probs ~ N(-36, 1); 4 epochs x 8 minibatches, entropy 0.01,
    hypernet 6 -> 256 -> F 256 with mo-humanoid6 dims (obs 45, act 12)."""
    import torch
    base = dict(BASE["c3"], N=4096, K=64, seed=3)
    cfg = mb.TrainConfig(**base)
    t = mb.Trainer(cfg)
    es, R, N, T = t.es, t.rows, cfg.N, cfg.T
    rng = np.random.default_rng(3)
    v = rng.normal(size=(N, T + 1, es.m))
    t.set("obs", rng.normal(size=(R, es.obs_dim)))
    t.set("action_pre", rng.normal(size=(R, es.act_dim)))
    t.set("logprob", rng.normal(-36.0, 1.0, size=R))
    t.set("reward", rng.normal(size=(R, es.m)))
    t.set("value", v[:, :T].reshape(R, es.m))
    t.set("next_value", v[:, 1:].reshape(R, es.m))
    t.set("terminated", rng.random(R) < 0.01)
    t.set("truncated", np.zeros(R, np.uint8))
    t.set("clusters", rng.dirichlet(np.ones(es.m), size=cfg.K))
    stream = torch.cuda.ExternalStream(mb.LIB.morlax_trainer_stream(t._h))

    def step(i):
        for ph in (5, 2, 3, 4):
            t.phase(i, ph)

    for i in range(3):
        step(i)
    ms = _events_ms(stream, lambda i: step(3 + i), 5)
    return {"workload": "config4-gae+ppo-update-4096env-T64-64pref", "metric": "transitions/s",
            "value": R / (ms / 1e3), "ms_per_step": ms}


# ---------------------------------------------------------------- roofline of the whole iteration
def iteration_roofline(prof, hbm_gbs, tflops, iter_ms):
    """roofline time per iteration = sum over phases of
    max(FLOP_phase / bf16 peak, bytes_phase / HBM peak), with the algorithmic
    FLOPs and bytes of every launch of the phase as the dataflow moves them
    (GEMM operand / activation / gradient images, theta and its packing,
    optimizer state, rollout batch writes) from the per-launch profile pass.
    frac = roofline time / measured time per iteration."""
    phases = {}
    for name, _ms, fl, by, _n in prof:
        ph = name.split("/")[0]
        f, b = phases.get(ph, (0.0, 0.0))
        phases[ph] = (f + fl, b + by)
    out, total = {}, 0.0
    for ph, (f, b) in phases.items():
        t_f = f / (tflops * 1e12) * 1e3
        t_b = b / (hbm_gbs * 1e9) * 1e3
        out[ph] = {"gflop": round(f / 1e9, 2), "gbytes": round(b / 1e9, 3), "ms_tensor": round(t_f, 4),
                   "ms_hbm": round(t_b, 4), "bound": "tensor" if t_f >= t_b else "hbm"}
        total += max(t_f, t_b)
    return {"roofline_ms": round(total, 4), "measured_ms": round(iter_ms, 4), "frac": total / iter_ms,
            "phases": out}


# ---------------------------------------------------------------- GPU arm
def self_launch(args):
    """--gpus N without a launcher: re-exec this script as N ranks under
    torch.distributed.run on this node (one process per GPU, NCCL)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(BASE))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-legs", action="store_true", help="skip the config 1 / 2 / 4 legs")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}: "
                         "launch one rank per GPU (torchrun --nproc-per-node N) or let bench.py self-launch")

    import torch
    import torch.distributed as dist

    import paper_2603_09237_b200 as mb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    base = dict(BASE[args.config])
    cfg = mb.TrainConfig(**{**base, "N": base["N"] * world, "K": base["K"] * world})
    nid = None
    if world > 1:
        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(mb.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        nid = bytes(buf.cpu().numpy().tobytes())
    trainer = mb.Trainer(cfg, world, rank, nid)
    stream = torch.cuda.ExternalStream(mb.LIB.morlax_trainer_stream(trainer._h))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for it in range(args.warmup):
        trainer.iteration(it)
    barrier()
    steps_per_iter = trainer.local_envs * cfg.T
    launches0 = trainer.kernel_launches
    # ---- timed region: CUDA events on the trainer's stream
    with Clocks(local) as clk:
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(args.steps):
            trainer.iteration(args.warmup + k)
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    launches = (trainer.kernel_launches - launches0) // args.steps
    # ---- e2e: host wall clock around the C-ABI call (H2D of sampled
    # preferences + minibatch indices and D2H of the stats inside each call)
    barrier()
    t0 = time.perf_counter()
    for k in range(args.steps):
        trainer.iteration(args.warmup + args.steps + k)
    barrier()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([ms, e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, e2e_s = float(tt[0]), float(tt[1])
    total_steps = world * steps_per_iter * args.steps
    value = total_steps / (ms / 1e3)
    e2e = total_steps / e2e_s
    # ---- per-kernel-class profile (separate pass, CUDA events per launch)
    import ctypes as C
    mb.LIB.morlax_trainer_profile_enable(trainer._h, 1)
    trainer.iteration(args.warmup + 2 * args.steps)
    n = mb.LIB.morlax_trainer_profile_count(trainer._h)
    prof = []
    for i in range(n):
        name = C.create_string_buffer(64)
        pm, pf, pb, pc = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
        mb.LIB.morlax_trainer_profile_get(trainer._h, i, name, C.byref(pm), C.byref(pf), C.byref(pb),
                                          C.byref(pc))
        prof.append((name.value.decode(), pm.value, pf.value, pb.value, pc.value))
    mb.LIB.morlax_trainer_profile_enable(trainer._h, 0)
    prof.sort(key=lambda x: -x[1])
    hbm, tflops, peak_src = peaks()
    top = prof[0]
    iter_ms = ms / args.steps
    iteration_roof = iteration_roofline(prof, hbm, tflops, iter_ms)
    if top[3] > 0 and top[2] == 0:
        ach = top[3] / (top[1] / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm}
    else:
        ach = top[2] / (top[1] / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": ach, "peak": tflops, "unit": "TFLOP/s",
                "frac": ach / tflops}
    traffic, tsrc = None, None
    kname = top[0].split("/")[-1]
    for tfile in ("r2_ncu_traffic.json", "r1_ncu_traffic.json"):  # the newest capture that has the kernel
        tpath = os.path.join(ROOT, "profiles", tfile)
        if traffic is None and os.path.exists(tpath):  # dram__bytes_read + write per launch, ncu --set full
            tj = json.load(open(tpath)).get(kname)
            if tj:
                traffic, tsrc = tj["dram_bytes_per_launch"], tj["capture"]
    roof.update({"traffic": traffic, "traffic_unit": "bytes/launch", "traffic_source": tsrc,
                 "algorithmic_bytes_per_launch": top[3] / top[4] if top[4] else None,
                 "kernel": kname, "class": top[0], "launches_per_iter": top[4],
                 "share_of_step": top[1] / sum(p[1] for p in prof),
                 "peak_source": peak_src + (" bf16 sustained" if roof["bound"] == "tensor" else " copy")})
    breakdown = {p[0]: {"ms": round(p[1], 3), "launches": p[4],
                        "tflops": round(p[2] / (p[1] / 1e3) / 1e12, 2) if p[2] else None,
                        "gbs": round(p[3] / (p[1] / 1e3) / 1e9, 1) if p[3] else None} for p in prof}
    # ---- Pareto leg (config 5: 1024 six-objective points, ref -1^6)
    pareto = None
    if rank == 0:
        rng = np.random.default_rng(4)
        w = rng.dirichlet(np.ones(6), size=1024)
        pts = w / np.linalg.norm(w, axis=1, keepdims=True) + rng.normal(0, 0.02, (1024, 6))
        mb.nondominated_mask(pts)
        t0 = time.perf_counter()
        mask = mb.nondominated_mask(pts)
        t1 = time.perf_counter()
        hv = mb.hypervolume_detailed(pts[mask.astype(bool)], -np.ones(6))
        t2 = time.perf_counter()
        hv_ex, _ = mb.hypervolume_exact(pts[mask.astype(bool)], -np.ones(6))
        t3 = time.perf_counter()
        pareto = {"points": 1024, "nondominated": int(mask.sum()), "mask_ms": round((t1 - t0) * 1e3, 3),
                  "hv_mc_ms": round((t2 - t1) * 1e3, 3), "hv": hv[0], "hv_stderr": hv[1],
                  "hv_samples": 1_000_000, "hv_exact": hv_ex, "hv_exact_ms": round((t3 - t2) * 1e3, 3)}
        try:  # the reference's own nondominated_filter / hypervolume_detailed (pareto.cpp:38-77, 209-277)
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            from pyoracle import Oracle
            r = Oracle("ref")
            t0 = time.perf_counter()
            rmask = r.nondominated_mask(pts)
            t1 = time.perf_counter()
            rhv = r.hypervolume_detailed(pts[rmask.astype(bool)], -np.ones(6))
            t2 = time.perf_counter()
            pareto["reference"] = {"mask_ms": round((t1 - t0) * 1e3, 3), "hv_mc_ms": round((t2 - t1) * 1e3, 3),
                                   "mask_equal": bool(np.array_equal(rmask, mask)),
                                   "hv_equal": bool(rhv[0] == hv[0] and rhv[1] == hv[1]), "threads": 1,
                                   "kind": "reference (oracle/_ref, Release flags)"}
        except Exception as ex:  # reported, never silently replaced
            pareto["reference"] = {"unavailable": str(ex)}
    # ---- CPU baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cores = os.cpu_count() or 1
            v, sample, secs = reference_sample(base, cores)
            cpu = {"value": v, "unit": "env-steps/s", "cores": cores, "kind": "reference",
                   "sample": sample, "sample_seconds": round(secs, 2)}
        except Exception as ex:  # reported, never silently replaced
            cpu = {"value": None, "unit": "env-steps/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {ex}"}
    legs = None
    if rank == 0 and world == 1 and not args.no_legs:
        legs = {"config1_pr1": leg_pr1(mb, not args.no_cpu_baseline), "config2": leg_c2(mb, peaks()[1]),
                "config4": leg_c4(mb)}
    es = mb.env_spec(cfg.env_name)
    slots = cfg.epochs * cfg.minibatch_count
    bmax = -(-cfg.N * cfg.T // cfg.minibatch_count)
    h2d = cfg.K * es.m * 4 + slots * (bmax + trainer.local_clusters + 1) * 4
    d2h = slots * 2 * 8 + 4 + trainer.local_envs * 12
    if rank == 0:
        print(json.dumps({
            "metric": "env-steps/s", "value": value, "unit": "env-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": iter_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16 (tcgen05 GEMMs, fp32 accumulate; fp32 env/elementwise, fp64 RNG transforms)",
            "data": "synthetic (seeded env rollouts; random-init hypernetworks)",
            "config": {"workload": WORKLOAD[args.config], "envs": cfg.N, "clusters": cfg.K, "T": cfg.T,
                       "env": cfg.env_name, "ppo": f"{cfg.epochs}x{cfg.minibatch_count}",
                       "parallelism": f"dp{world}", "l2": "working set > L2 (Adam state 666 MB/iter)"},
            "e2e": {"value": e2e, "unit": "env-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches, "roofline": {**roof, "iteration_frac": iteration_roof["frac"],
                                                   "iteration": iteration_roof},
            "cpu_baseline": cpu, "clocks": clk.summary(),
            "breakdown_ms_per_iter": breakdown, "pareto": pareto, "other_configs": legs,
        }))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
