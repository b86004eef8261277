#!/usr/bin/env python
"""Benchmark of the RaDe-GS rasterizer hot path on B200 (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--views-per-step B]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...        # the fp64 CPU oracle arm (rank 0 only)

A step = B views per rank, each view one pass of the whole hot path:
rd_preprocess → rd_bin → rd_render_fwd → rd_render_bwd (gradients accumulated into one
flat buffer), then — for N > 1 — one NCCL all-reduce (sum) of the flat gradient buffer
(the only exchange step, §8(e)). Views are partitioned across ranks (v mod N = rank) with
the Gaussians replicated: weak scaling. `value` = views processed by all ranks / the max
over ranks of the device-timed region (CUDA events, barrier + synchronize on both sides).

Prints ONE JSON line on rank 0 (see DESIGN.md §Measurement for every key).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
from concurrent.futures import ThreadPoolExecutor
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd frames/sec (color+depth+normal)"
UNIT = "frames/s"
SEED_COT = 1000

# ----------------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() in ("active", "1"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- roofline model


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    hbm = d.get("hbm_gbs", 6650.0)
    src = "measured" if "hbm_gbs" in d else "fallback"
    sm_mhz = d.get("sm_max_mhz", 1965.0)
    return hbm, src, sm_mhz


def fp32_peak_tflops(n_sm, sm_mhz):
    """FP32 FFMA peak: the measured one (profiles/fp32_peak.json, tools/ffma_peak.cu on this
    pool's B200s); else the formula SMs × 128 FP32 lanes × 2 flop × clock. Returns (TFLOP/s,
    source)."""
    p = os.path.join(ROOT, "profiles", "fp32_peak.json")
    if os.path.exists(p):
        return float(json.load(open(p))["fp32_ffma_tflops"]), "measured FFMA (profiles/fp32_peak.json)"
    return n_sm * 128 * 2 * sm_mhz * 1e6 / 1e12, f"formula: {n_sm} SMs x 128 lanes x 2 flop x {sm_mhz:.0f} MHz"


# algorithmic work per unit: SURVEY.md §8(d)'s units
FWD_FLOP_PASS = 46     # K3: flop per α-passing (blended) pair: 23 FP32-pipe instructions, FFMA = 2
BWD_FLOP_PASS = 120    # K4: flop per α-passing pair
K1_B_ALL, K1_B_VIS = 12, 300               # K1: cull read per Gaussian / 224 B in + 76 B out per visible
K5_B_VIS = 600                             # K5: params 236 + 2-D grads 60 + record 64 + grads 236 per visible
# batched K5 (rd_preprocess_bwd_views): per Gaussian visible in any view of the batch its SH row
# once (192 B) and its SH gradient row reduced once (read + write, 384 B); per (visible Gaussian,
# view) the geometry pass: parameters 56 B (means, scales, rotation, opacity), the 80-B 2-D
# gradient row and the geometry gradient rows reduced (read + write, 88 B); the views'
# tiles_touched (4 B per Gaussian per view)
K5V_B_UNION, K5V_B_VIS, K5V_B_ALL = 576, 224, 4


def kernel_work(name, t, views, tile_passes):
    """Algorithmic (bytes or flops, bound) summed over the timed views for one kernel."""
    n, nvis, M = t["n"], t["n_visible"], t["n_duplicates"]
    if name == "preprocess_fwd":
        return K1_B_ALL * n * views + K1_B_VIS * nvis, "hbm"
    if name == "depth_sort":   # K2h: key per Gaussian + rect per visible; pass 0: key per Gaussian
        # read, (key, id) per visible written; passes 1-3: (key, id) read + written per visible
        return 8 * n * views + (8 + 8 + 3 * 16) * nvis, "hbm"
    if name == "scan":         # sorted id + gathered count read, offset written, per visible
        return 12 * nvis, "hbm"
    if name == "duplicate":    # K2c + first tile pass: offsets, sorted ids, rects of the visible,
        return 16 * nvis + 8 * M, "hbm"  # (tile, id) 8 B written per duplicate
    if name == "tile_sort":    # the remaining tile passes: (tile, id) 8 B read + 8 B written
        return 16 * M * (tile_passes - 1), "hbm"
    if name == "ranges":
        return 4 * M, "hbm"
    if name == "render_fwd":
        return FWD_FLOP_PASS * t["pairs_blended_fwd"], "alu"
    if name == "render_bwd":
        return BWD_FLOP_PASS * t["pairs_blended_fwd"], "alu"
    if name == "preprocess_bwd":
        if t.get("n_visible_union"):  # batched K5
            return K5V_B_UNION * t["n_visible_union"] + K5V_B_VIS * nvis + K5V_B_ALL * n * views, "hbm"
        return K5_B_VIS * nvis, "hbm"
    raise KeyError(name)


# ----------------------------------------------------------------------------- distributed


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_if_needed(args):
    """`python bench.py --gpus N` (N > 1) without a torchrun environment re-launches itself
    as N ranks under torch.distributed.run on this node (127.0.0.1 rendezvous) and returns
    the launcher's exit code; None when this process is already a rank (or N = 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def views_per_step(args, n_views, ws):
    """--views-per-step B (views per rank per step), or 'epoch': B = ceil(V/P), one all-reduce
    per pass over the config's views."""
    if str(args.views_per_step) == "epoch":
        return max(1, math.ceil(n_views / ws))
    b = int(args.views_per_step)
    if b < 1:
        raise SystemExit("--views-per-step must be >= 1 or 'epoch'")
    return b


def barrier(dist_on):
    if dist_on:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, dist_on, device):
    if not dist_on:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- CPU oracle arm


def oracle_frame_time(scene, cam, opt, n_pix=16, n_grad=1, seed=0):
    """Times the oracle as it stands on a bounded sample of one view: the forward on n_pix
    random pixels and the dual-number gradient of n_grad random visible Gaussians; returns
    (seconds per full frame fwd+bwd extrapolated, description, cores)."""
    import oracle
    rng = np.random.default_rng(seed)
    W, H = cam.width, cam.height
    pix = rng.choice(W * H, n_pix, replace=False)
    tf = np.zeros(3)
    oracle.render(scene, cam, opt, pixels=pix, timing=tf)
    n_vis = int(tf[2])
    # pick visible (in-front, near-centre) Gaussians with small footprints as the gradient sample
    x = (np.asarray(cam.R, np.float64) @ scene.means.astype(np.float64) + np.asarray(cam.t, np.float64)[:, None])
    z = x[2]
    u = cam.fx * x[0] / np.maximum(z, 1e-6) + cam.cx
    v = cam.fy * x[1] / np.maximum(z, 1e-6) + cam.cy
    ok = (z > 0.5) & (u > 0) & (u < W) & (v > 0) & (v < H) & (scene.opacities > 0.05)
    cand = np.nonzero(ok)[0]
    gids = rng.choice(cand, min(n_grad, len(cand)), replace=False) if len(cand) else np.zeros(0, np.int64)
    cot = {"color": np.zeros((3, H, W)), "depth": np.zeros((H, W)), "normal": np.zeros((3, H, W)),
           "alpha": np.zeros((H, W))}
    r = np.random.default_rng(seed + 1)
    cot["color"][:] = r.normal(size=(3, H, W))
    cot["depth"][:] = r.normal(size=(H, W))
    tg = np.zeros(3)
    if len(gids):
        oracle.grad(scene, cam, opt, cot, gids, timing=tg)
    t_fwd = tf[0] + tf[1] * (W * H / n_pix)
    t_bwd = tg[0] + tg[1] * (n_vis / max(len(gids), 1))
    desc = (f"one view of the workload: fp64 forward on {n_pix} random pixels (of {W * H}) + dual-number gradient "
            f"of {len(gids)} visible Gaussian(s) (of {n_vis}), extrapolated to the full frame; "
            f"measured {tf[0] + tf[1] + tg[0] + tg[1]:.1f} s")
    return t_fwd + t_bwd, desc, oracle.num_threads(), tf[0] + tf[1] + tg[0] + tg[1]


def run_reference(args, cfg_name, config):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    import scenegen as sg
    oracle.build()
    scene, cams, opt = sg.config_scene_and_cameras(cfg_name, n_gaussians=args.n_gaussians)
    times, desc, cores = [], "", 1
    for step in range(args.warmup + args.steps):
        cam = cams[step % len(cams)]
        t, desc, cores, _ = oracle_frame_time(scene, cam, opt, n_pix=args.ref_pixels, n_grad=args.ref_grads,
                                              seed=step)
        if step >= args.warmup:
            times.append(t)
    frame_s = float(np.mean(times))
    value = 1.0 / frame_s
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": frame_s * 1e3 * views_per_step(args, len(cams), 1),
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"each step: {desc}"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- gloo dry run


def run_dry_gloo(args, cfg_name, config):
    """The GPU arm's distributed skeleton on CPU: the same rank layout (torchrun env), view
    partition, views per step (incl. 'epoch'), flat-buffer accumulation, bucketed all-reduce,
    barrier + max-over-ranks timing and rank-0 JSON line — with each view's fwd+bwd replaced by
    a deterministic fake gradient (the CUDA path needs a GPU). Checks after every step that
    the all-reduced buffer equals the sum of the fake gradients of ALL ranks' views of the
    step and that the replicas agree bitwise."""
    import torch
    import torch.distributed as dist
    import scenegen as sg
    from paper_2406_01467_b200.parallel import FlatGrads, views_for_rank

    ws, rank, _ = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    dist_on = ws > 1
    if dist_on:
        dist.init_process_group("gloo")
    n_views = sg.CONFIGS[cfg_name]["views"]
    n = 257  # fake Gaussians (the buffer layout of FlatGrads, small)
    fg = FlatGrads.allocate(n, 16, "cpu")
    B = views_per_step(args, n_views, ws)
    mine = views_for_rank(n_views, ws, rank) or [rank % n_views]  # more ranks than views: repeat one

    def fake(v):
        return torch.full((fg.flat.numel(),), float(v % 7 + 1)) * (torch.arange(fg.flat.numel()) % 5 + 1)

    counter = {"v": 0}

    def step():
        fg.zero_()
        ks = []
        for _ in range(B):
            ks.append(counter["v"])
            counter["v"] += 1
        for k in ks:
            fg.flat += fake(mine[k % len(mine)])
        fg.allreduce(bucket_bytes=args.bucket_mb << 20)
        # every rank's views of this step: rank r ran views_for_rank(...)[k % len] for the same ks
        exp = torch.zeros_like(fg.flat)
        for r in range(ws):
            vr = views_for_rank(n_views, ws, r) or [r % n_views]
            for k in ks:
                exp += fake(vr[k % len(vr)])
        assert torch.equal(fg.flat, exp), "all-reduced buffer != sum over ranks"
        if dist_on:
            cs = torch.tensor([float(fg.flat.double().sum())], dtype=torch.float64)
            lo, hi = cs.clone(), cs.clone()
            dist.all_reduce(lo, op=dist.ReduceOp.MIN)
            dist.all_reduce(hi, op=dist.ReduceOp.MAX)
            assert lo.item() == hi.item(), "replicas differ"

    for _ in range(args.warmup):
        step()
    barrier(dist_on)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    barrier(dist_on)
    elapsed = time.perf_counter() - t0
    if dist_on:
        t = torch.tensor([elapsed], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    total = args.steps * B * ws
    config.update({"views_per_step_per_rank": B, "parallelism": f"view-parallel dp{ws} (gloo dry run)"})
    line = {"metric": METRIC, "value": total / elapsed, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config,
            "dry_run": "gloo: fake per-view gradients, all-reduce checked against the sum over ranks", "gpu_launches": 0}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist_on:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- GPU arm


def run_gpu(args, cfg_name, config):
    import torch
    import paper_2406_01467_b200 as P
    import scenegen as sg

    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws} (launch with torchrun, or let "
                         f"bench.py re-launch itself by leaving WORLD_SIZE unset)")
    dist_on = ws > 1 or args.nccl_single
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if dist_on:
        import torch.distributed as dist
        if ws == 1:  # --nccl-single: the N > 1 code path (NCCL group, side-stream bucketed
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")  # all-reduce, barriers, max over
            os.environ.setdefault("MASTER_PORT", str(_free_port()))  # ranks) as one rank
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=device)

    from paper_2406_01467_b200.parallel import FlatGrads, views_for_rank

    scene, cams, opt = sg.config_scene_and_cameras(cfg_name, n_gaussians=args.n_gaussians)
    n = scene.n
    my_views = [cams[v] for v in (views_for_rank(len(cams), ws, rank) or [rank % len(cams)])]
    B = views_per_step(args, len(cams), ws)
    comm_stream = torch.cuda.Stream(device) if dist_on else None  # the all-reduce's side stream
    g = P.Gaussians.from_numpy(scene, device)
    K = g.sh.shape[1]
    fg = FlatGrads.allocate(n, K, device)  # one flat buffer: the all-reduce operand
    grads = fg.as_gaussians()
    H, W = cams[0].height, cams[0].width
    n_ring = min(B * 2, 8)
    gen = torch.Generator(device=device)
    gen.manual_seed(SEED_COT + rank)
    cots = [torch.randn((10, H, W), generator=gen, device=device, dtype=torch.float32) for _ in range(n_ring)]
    opts = dict(tile=args.tile, alpha_min=opt.alpha_min, alpha_max=opt.alpha_max, T_min=opt.T_min,
                median_T=opt.median_T, dilation=opt.dilation, bg=opt.bg, sh_degree=opt.sh_degree,
                guard_band=opt.guard_band if args.guard_band is None else args.guard_band)
    config["guard_band"] = opts["guard_band"]
    # Views are pipelined over `args.pipeline` CUDA streams, each with its own rd_view and
    # output maps (and its own host thread): the views of a step run concurrently. Their
    # gradient accumulations (K5, rd_preprocess_bwd) add into the one flat buffer with L2
    # reductions, so they need no mutual order.
    if args.pipeline <= 0:  # every view of a step on its own stream: they all start at once
        args.pipeline = min(max(1, B), 8)
    P_ = max(1, args.pipeline)
    slots = []
    lo_prio, hi_prio = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
    config["stream_priorities"] = args.prio
    for i in range(P_):
        # --prio views: slot i at priority hi + i (clamped to the device's range; lower = higher)
        st = torch.cuda.Stream(device, priority=min(lo_prio, hi_prio + i) if args.prio != "none" else 0)
        with torch.cuda.stream(st):  # the view's scratch is allocated on its own stream
            slot = {"stream": st, "view": P.View(device),
                    # the maps are planes of one [10, H, W] buffer: one D2H copy per view (e2e)
                    "outbuf": torch.empty((10, H, W), device=device),

                    "cot": torch.empty((10, H, W), device=device),
                    "done": torch.cuda.Event(),
                    # --stagger: recorded after the view's rd_bin; set on the host once recorded
                    "binned": torch.cuda.Event(), "binned_host": threading.Event()}
            ob = slot["outbuf"]
            slot["outs"] = {"color": ob[0:3], "depth": ob[3], "normal": ob[4:7], "alpha": ob[7],
                            "distortion": ob[8], "consistency": ob[9]}
        slots.append(slot)
    view = slots[0]["view"]
    outs = slots[0]["outs"]
    streams = {"k5": torch.cuda.Stream(device, priority=hi_prio if args.prio == "views-k5" else 0),  # the batched K5
               "zero": torch.cuda.Stream(device),  # the step's gradient zeroing
               "k1": torch.cuda.Stream(device)}  # --k1 batched: the round's K1
    k1_ev = torch.cuda.Event()
    zeroed = {"ev": torch.cuda.Event()}
    k5_done = torch.cuda.Event()
    counter = {"v": 0}
    main_stream = torch.cuda.current_stream(device)

    phase_log = [] if os.environ.get("RADE_PHASES") else None

    def one_view(slot, cam, cot, io=None):
        """io (end-to-end pass): events that order the view's forward after the D2H of the
        slot's previous maps, publish the forward for its D2H, hold K4 until the H2D of the
        cotangents landed, and publish K4 (the cotangent buffer is free again). K5 adds the
        view's gradients with L2 reductions, so the views' K5 calls need no mutual order."""
        st, vw, o = slot["stream"], slot["view"], slot["outs"]
        ph = [] if phase_log is not None else None  # diagnostics: per-view phase events

        def mark():
            if ph is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                ph.append(e)
        with torch.cuda.stream(st):
            prev = slot.get("stagger_after")
            if prev is not None:  # --stagger S: start once the view S slots earlier is binned
                prev["binned_host"].wait()
                st.wait_event(prev["binned"])
            mark()
            if slot.get("k1_done") is not None:  # --k1 batched: the round's K1 ran in one launch
                st.wait_event(slot["k1_done"])
            else:
                P.rd_preprocess(vw, g, cam, opts, stream=st)
            mark()  # K1 done
            P.rd_bin(vw, stream=st)
            if args.stagger:
                slot["binned"].record(st)
                slot["binned_host"].set()
            mark()
            if io:
                st.wait_event(io["outs_free"])
            if args.distortion:  # NEXT-1: + the depth-distortion map and its gradient
                mark()
                P.rd_render_fwd_ex(vw, o["color"], o["depth"], o["normal"], o["alpha"], o["distortion"], stream=st)
            else:
                mark()
                P.rd_render_fwd(vw, o["color"], o["depth"], o["normal"], o["alpha"], stream=st)
            mark()
            if args.normal_consistency:  # NEXT-2: L_n on the maps (its plane is read back with them)
                P.rd_normal_consistency(cam, o["depth"], o["alpha"], o["normal"], consistency=o["consistency"],
                                        stream=st)
            if io:
                io["fwd_done"].record(st)  # every map plane of the view is written
                st.wait_event(io["cot_ready"])
                if io.get("loss_fn") is not None:  # e2e loss mode: cotangents from the loss on device
                    cot = io["loss_fn"](o)
            if args.normal_consistency:  # its cotangents join the maps'
                ct = slot["cot"]
                ct.copy_(cot)
                P.rd_normal_consistency_bwd(cam, o["depth"], o["normal"], ct[9], ct[3], ct[7], ct[4:7], stream=st)
                cot = ct
            if args.distortion:
                P.rd_blend_bwd_ex(vw, cot[0:3], cot[3], cot[4:7], cot[7], cot[8], stream=st)
            else:
                P.rd_blend_bwd(vw, cot[0:3], cot[3], cot[4:7], cot[7], stream=st)  # K4: view-private output
            if io:
                io["k4_done"].record(st)
            mark()
            if args.k5 in ("per-view", "split", "split-set"):
                st.wait_event(zeroed["ev"])  # the step's gradients are zeroed
            if args.k5 == "per-view":
                P.rd_preprocess_bwd(vw, g, grads, stream=st)  # K5: += by L2 reductions
            elif args.k5 in ("split", "split-set"):  # K5 geometry now, overlapping the other views' K3/K4
                P.rd_preprocess_bwd_geometry(vw, g, grads, stream=st)
            slot["done"].record(st)  # batched K5: the round's rd_preprocess_bwd_views waits for this
            mark()
        if ph is not None:
            phase_log.append(ph)

    pool = ThreadPoolExecutor(max_workers=max(1, args.pipeline)) if args.host_threads else None

    def cam_of(k):
        return my_views[k % len(my_views)]

    def run_views(per_view):
        """Zero the gradients, run B views through the slots, join, all-reduce.
        With host threads (default) each slot's views are issued by their own host thread, so
        one view's rd_bin (which waits for its count of duplicates) does not hold
        back the issue of the other slots' views."""
        start = torch.cuda.Event()
        start.record(main_stream)  # the previous step is complete (its K5 / all-reduce)
        for sl in slots:
            sl["stream"].wait_event(start)
        # the gradients are written by K5 only, so their zeroing (a 354-MB memset at C3) runs on
        # its own stream beside the views' K1..K4; every K5 waits for it
        zs = streams["zero"]
        zs.wait_event(start)
        with torch.cuda.stream(zs):
            if args.k5 in ("set", "split-set"):  # the first round's K5 sets the SH rows (RD_K5_SET_SH)
                fg.zero_geometry_()
            else:
                fg.zero_()
        zeroed["ev"].record(zs)
        ks = []
        for b in range(B):
            ks.append(counter["v"])
            counter["v"] += 1
        # rounds of one view per slot; with the batched K5 (default) each round ends with ONE
        # rd_preprocess_bwd_views over its views on k5_stream (after every view's K4), and a
        # slot's next view waits for it (its K1 rewrites the view's 2-D gradient rows)
        last = []
        for r0 in range(0, len(ks), P_):
            rnd = ks[r0:r0 + P_]
            used = [slots[i] for i in range(len(rnd))]
            if args.k1 == "batched":  # one K1 launch for the round's views (rd_preprocess_views)
                k1s = streams["k1"]
                k1s.wait_event(start)
                if r0 > 0:
                    k1s.wait_event(k5_done)  # the previous round's K5 has read the views' 2-D gradients
                # --k1-groups G: the round's views in G batched K1 launches, so the first group's
                # views start binning while the next group's K1 runs
                ng = max(1, min(args.k1_groups, len(used)))
                per = (len(used) + ng - 1) // ng
                for gi in range(0, len(used), per):
                    grp, gk = used[gi:gi + per], rnd[gi:gi + per]
                    P.rd_preprocess_views([sl["view"] for sl in grp], g, [cam_of(k) for k in gk], opts, stream=k1s)
                    ev = k1_ev if gi == 0 else torch.cuda.Event()
                    ev.record(k1s)
                    for sl in grp:
                        sl["k1_done"] = ev
            else:
                for sl in used:
                    sl["k1_done"] = None
            for i, sl in enumerate(used):
                sl["binned_host"].clear()
                sl["stagger_after"] = used[i - args.stagger] if args.stagger and i >= args.stagger else None
            if pool is None:
                for sl, k in zip(used, rnd):
                    per_view(sl, k)
            else:
                def worker(sl, k):
                    torch.cuda.set_device(device)  # per thread
                    per_view(sl, k)

                futs = [pool.submit(worker, sl, k) for sl, k in zip(used, rnd)]
                for f in futs:
                    f.result()
            if args.k5 in ("batched", "split", "set", "split-set"):
                k5s = streams["k5"]
                k5s.wait_event(zeroed["ev"])
                for sl in used:
                    k5s.wait_event(sl["done"])
                if args.k5 == "split":  # the round's SH part (its geometry parts ran per view)
                    P.rd_preprocess_bwd_views_sh([sl["view"] for sl in used], g, grads, stream=k5s)
                elif args.k5 == "split-set":  # the round's SH part, setting the rows in the first round
                    P.rd_preprocess_bwd_views_ex([sl["view"] for sl in used], g, grads,
                                                 flags=P.rade.RD_K5_SH_ONLY | (P.rade.RD_K5_SET_SH if r0 == 0 else 0),
                                                 stream=k5s)
                elif args.k5 == "set":  # the step's first round SETS the SH gradient rows
                    P.rd_preprocess_bwd_views_ex([sl["view"] for sl in used], g, grads,
                                                 flags=P.rade.RD_K5_SET_SH if r0 == 0 else 0, stream=k5s)
                else:
                    P.rd_preprocess_bwd_views([sl["view"] for sl in used], g, grads, stream=k5s)
                k5_done.record(k5s)
                for sl in used:
                    sl["stream"].wait_event(k5_done)
                last = [k5_done]
            else:
                last = [sl["done"] for sl in used]
        waiter = main_stream if comm_stream is None else comm_stream
        for ev in last:
            waiter.wait_event(ev)
        if comm_stream is not None:  # NCCL sum over ranks on a side stream once every view's K5 has added its rows
            with torch.cuda.stream(comm_stream):
                fg.allreduce(bucket_bytes=args.bucket_mb << 20)
            main_stream.wait_stream(comm_stream)

    def step():
        run_views(lambda sl, k: one_view(sl, my_views[k % len(my_views)], cots[k % n_ring]))

    # ---------------- device-resident timed region (no per-kernel events: pipelined streams)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    barrier(dist_on)
    torch.cuda.synchronize()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e0.record()
    for j in range(args.steps):
        step()
        marks[j].record()  # step boundary on the main stream (it waited for the step's last K5)
    e1.record()
    torch.cuda.synchronize()
    barrier(dist_on)
    clk = clocks.stop()
    elapsed_ms = max_over_ranks(e0.elapsed_time(e1), dist_on, device)
    total_views = args.steps * B * ws
    value = total_views / (elapsed_ms / 1e3)
    step_ms = np.array([e0.elapsed_time(marks[0])] + [marks[j - 1].elapsed_time(marks[j]) for j in range(1, args.steps)])
    views_covered = len(set((k % len(my_views)) for k in range(args.warmup * B, (args.warmup + args.steps) * B)))

    if os.environ.get("RADE_PROF_CONC"):  # diagnostics: per-kernel times under the concurrent schedule
        for sl in slots:
            P.rd_set_profiling(sl["view"], True)
        torch.cuda.synchronize()
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        acc = {}
        for sl in slots:
            t = P.rd_get_timings(sl["view"], reset=True)
            P.rd_set_profiling(sl["view"], False)
            for k, v in t["ms"].items():
                acc[k] = acc.get(k, 0.0) + v / max(t["views"], 1) / len(slots)
        print("concurrent per-kernel ms per view:", {k: round(v, 4) for k, v in acc.items()}, flush=True)
    if phase_log:  # diagnostics: [start, K1 done, binned, fwd start, fwd end, K4 end, K5 end] per view, ms
        t0e = phase_log[-4 * 5][0] if len(phase_log) >= 20 else phase_log[0][0]
        rows = [[t0e.elapsed_time(e) for e in ph] for ph in phase_log[-20:]]
        json.dump(rows, open(os.environ["RADE_PHASES"], "w"))
        phase_log.clear()

    # ---------------- per-kernel timings: the same steps again, serialised on one stream with
    # the ABI's CUDA-event hooks around every kernel (rd_set_profiling)
    # every slot keeps its view and buffers, but all of them (and the batched K5) run on one
    # stream from one host thread, so the kernels are serialised and each one's CUDA-event time
    # is its own; timings are summed over the slots' views
    prof_stream = torch.cuda.Stream(device)
    saved = [sl["stream"] for sl in slots], streams["k5"], pool, streams["zero"], streams["k1"]
    for sl in slots:
        sl["stream"] = prof_stream
        P.rd_set_profiling(sl["view"], True)
    streams["k5"], streams["zero"], streams["k1"], pool = prof_stream, prof_stream, prof_stream, None
    torch.cuda.synchronize()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    tim = None
    for sl in slots:
        t = P.rd_get_timings(sl["view"], reset=True)
        P.rd_set_profiling(sl["view"], False)
        if tim is None:
            tim = t
            continue
        for key in ("ms", "launches"):
            for kname, val in t[key].items():
                tim[key][kname] = tim[key].get(kname, 0) + val
        for key in ("n_duplicates", "views", "pairs_evaluated_fwd", "pairs_blended_fwd", "pairs_evaluated_bwd",
                    "n_visible", "n_visible_union", "pairs_issued_fwd"):
            tim[key] += t[key]
        for kname, val in t["n_culled"].items():
            tim["n_culled"][kname] += val
    for sl, st_ in zip(slots, saved[0]):
        sl["stream"] = st_
    streams["k5"], pool, streams["zero"], streams["k1"] = saved[1], saved[2], saved[3], saved[4]

    # ---------------- end-to-end: per step, inputs from pinned host memory in, result out.
    # loss mode (default): a view's input is its ground-truth RGB image (uint8, the training
    # data), the user-side loss (L1 colour, plus the regularisers' weights when enabled) and its
    # cotangents are computed on the device with torch ops, and the step's result read back is
    # the loss (4 B per view). maps mode: 8-channel fp32 cotangent images in, the rendered map
    # planes out (a loss computed on the host; PCIe-bound).
    e2e = None
    if not args.no_e2e and args.e2e_mode == "loss":
        gen_gt = torch.Generator()
        gen_gt.manual_seed(SEED_COT + 7 + rank)
        host_gts = [torch.randint(0, 256, (3, H, W), generator=gen_gt, dtype=torch.uint8).pin_memory()
                    for _ in range(n_ring)]
        dev_gts = [torch.empty((3, H, W), dtype=torch.uint8, device=device) for _ in slots]
        host_loss = [torch.zeros(1, dtype=torch.float32).pin_memory() for _ in slots]
        dev_loss = [torch.zeros(1, dtype=torch.float32, device=device) for _ in slots]
        cot_bufs = [torch.zeros((10, H, W), device=device) for _ in slots]
        cins = [torch.cuda.Stream(device) for _ in slots]
        couts = [torch.cuda.Stream(device) for _ in slots]
        ios = [{k: torch.cuda.Event() for k in ("cot_ready", "k4_done", "fwd_done", "outs_free", "loss_done")}
               for _ in slots]
        lam_d, lam_n = 100.0 / (H * W), 0.05 / (H * W)  # regulariser weights (RaDe-GS-like magnitudes)
        h2d = d2h = 0
        io_lock = threading.Lock()

        def make_loss_fn(i):
            def loss_fn(o):
                cb = cot_bufs[i]
                diff = o["color"] - dev_gts[i].float() * (1.0 / 255.0)
                dev_loss[i].copy_(diff.abs().mean().reshape(1))
                torch.sign(diff, out=cb[0:3])
                cb[0:3].mul_(1.0 / (3 * H * W))
                if args.distortion:
                    cb[8].fill_(lam_d)
                if args.normal_consistency:
                    cb[9].fill_(lam_n)
                ios[i]["loss_done"].record(torch.cuda.current_stream(device))
                return cb
            return loss_fn

        for i in range(len(slots)):
            ios[i]["loss_fn"] = make_loss_fn(i)

        def per_view_loss(sl, k):
            nonlocal h2d, d2h
            i = slots.index(sl)
            io = ios[i]
            with torch.cuda.stream(cins[i]):
                cins[i].wait_event(io["k4_done"])  # the slot's previous loss has read the image
                dev_gts[i].copy_(host_gts[k % n_ring], non_blocking=True)
                io["cot_ready"].record(cins[i])
            one_view(sl, my_views[k % len(my_views)], None, io)
            with torch.cuda.stream(couts[i]):
                couts[i].wait_event(io["loss_done"])
                host_loss[i].copy_(dev_loss[i], non_blocking=True)
                io["outs_free"].record(couts[i])
            with io_lock:
                h2d += dev_gts[i].numel()
                d2h += 4

        steps_e2e = max(1, args.steps)
        run_views(per_view_loss)
        torch.cuda.synchronize()
        h2d = d2h = 0
        barrier(dist_on)
        t0 = time.perf_counter()
        for _ in range(steps_e2e):
            run_views(per_view_loss)
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(time.perf_counter() - t0, dist_on, device)
        e2e = {"value": steps_e2e * B * ws / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d // steps_e2e,
               "d2h_bytes_per_step": d2h // steps_e2e, "mode": "loss",
               "what": "per view: H2D of the view's ground-truth RGB image (uint8) from pinned host memory, the "
                       "ABI calls, the user-side L1 colour loss and its cotangent on the device (torch), D2H of the "
                       "loss; batched K5 per round; Gaussians and gradients stay resident (model state); host wall "
                       "clock, max over ranks",
               "last_loss": float(host_loss[0].item())}
    if not args.no_e2e and args.e2e_mode == "maps":
        nch = 10 if args.normal_consistency else 9 if args.distortion else 8  # cotangent channels consumed
        host_cots = [c[:nch].cpu().pin_memory() for c in cots]
        h2d = 0
        d2h = 0
        n_out = 10 if args.normal_consistency else 9 if args.distortion else 8  # map planes read back
        host_outs = [torch.empty((n_out, H, W), dtype=torch.float32).pin_memory() for _ in slots]
        dev_cots = [torch.empty((nch, H, W), device=device) for _ in slots]

        # transfers on their own copy streams, overlapped with the compute of other views:
        # the H2D of a view's cotangents is only awaited by its K4, the D2H of its maps only
        # by the next forward of the same slot
        cins = [torch.cuda.Stream(device) for _ in slots]   # per slot: its host thread owns them
        couts = [torch.cuda.Stream(device) for _ in slots]
        io_lock = threading.Lock()
        ios = [{k: torch.cuda.Event() for k in ("cot_ready", "k4_done", "fwd_done", "outs_free")} for _ in slots]

        tl_path = os.environ.get("RADE_E2E_TIMELINE")  # diagnostics: per-view event timeline
        tl = []

        def tev(stream):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            return e

        def per_view_e2e(sl, k):
            nonlocal h2d, d2h
            i = slots.index(sl)
            io = ios[i]
            cin, cout = cins[i], couts[i]
            rec = {"host": time.perf_counter()} if tl_path else None
            with torch.cuda.stream(cin):
                cin.wait_event(io["k4_done"])  # the slot's previous K4 has read the buffer
                if rec is not None:
                    rec["h2d0"] = tev(cin)
                dev_cots[i].copy_(host_cots[k % n_ring], non_blocking=True)
                io["cot_ready"].record(cin)
                if rec is not None:
                    rec["h2d1"] = tev(cin)
            with io_lock:
                h2d += dev_cots[i].numel() * 4
            if rec is not None:
                rec["v0"] = tev(sl["stream"])
            one_view(sl, my_views[k % len(my_views)], dev_cots[i], io)
            if rec is not None:
                rec["v1"] = tev(sl["stream"])
                rec["host_end"] = time.perf_counter()
            with torch.cuda.stream(cout):
                cout.wait_event(io["fwd_done"])
                if rec is not None:
                    rec["d2h0"] = tev(cout)
                t = sl["outbuf"][:n_out]
                host_outs[i].copy_(t, non_blocking=True)
                with io_lock:
                    d2h += t.numel() * 4
                io["outs_free"].record(cout)
                if rec is not None:
                    rec["d2h1"] = tev(cout)
            if rec is not None:
                tl.append(rec)

        def step_e2e():
            run_views(per_view_e2e)

        steps_e2e = max(1, args.steps)
        step_e2e()
        torch.cuda.synchronize()
        h2d = d2h = 0
        barrier(dist_on)
        t0 = time.perf_counter()
        for _ in range(steps_e2e):
            step_e2e()
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(time.perf_counter() - t0, dist_on, device)
        if tl_path and tl:
            base_e, base_h = tl[0]["h2d0"], tl[0]["host"]
            rows = [{k: (base_e.elapsed_time(v) if isinstance(v, torch.cuda.Event) else (v - base_h) * 1e3)
                     for k, v in r.items()} for r in tl]
            json.dump(rows, open(tl_path, "w"), indent=0)
        e2e = {"value": steps_e2e * B * ws / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d // steps_e2e,
               "d2h_bytes_per_step": d2h // steps_e2e, "mode": "maps",
               "what": "per view: H2D of the view's cotangent image (8 channels, 9 with --distortion, 10 with "
                       "--normal-consistency) from pinned host memory, the five C-ABI calls, one D2H of the rendered "
                       "map planes, on the view's own copy streams overlapped with the other views' compute; "
                       "Gaussians and gradients stay resident (model state); host wall clock, max over ranks"}

    # ---------------- roofline of the dominant kernel + per-kernel breakdown
    hbm, hbm_src, sm_max = peaks()
    n_sm = torch.cuda.get_device_properties(device).multi_processor_count
    fp32, fp32_src = fp32_peak_tflops(n_sm, sm_max)
    views_timed = tim["views"]
    tim_ext = dict(tim)
    tim_ext["n"] = n
    st = P.rd_view_stats(view)
    tile_passes = (2 if st["tiles_x"] > 256 else 1) + (2 if st["tiles_y"] > 256 else 1)
    kernels = {}
    for name, ms in tim["ms"].items():
        launches = tim["launches"][name]
        if launches == 0:
            continue
        work, bound = kernel_work(name, tim_ext, views_timed, tile_passes)
        avg_ms = ms / launches
        per_launch = work / launches
        if bound == "hbm":
            ach = per_launch / (avg_ms * 1e-3) / 1e9
            kernels[name] = {"ms_per_launch": avg_ms, "share": None, "bound": "hbm", "achieved": ach,
                             "unit": "GB/s", "frac": ach / hbm}
        else:
            ach = per_launch / (avg_ms * 1e-3) / 1e12
            kernels[name] = {"ms_per_launch": avg_ms, "share": None, "bound": "alu", "achieved": ach,
                             "unit": "TFLOP/s", "frac": ach / fp32}
    tot_ms = sum(tim["ms"].values())
    for name in kernels:
        kernels[name]["share"] = tim["ms"][name] / tot_ms
    dom = max(kernels, key=lambda k: tim["ms"][k])
    dk = kernels[dom]
    traffic, issue, capture = None, None, None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        tr = json.load(open(tr_path)).get(dom)
        if isinstance(tr, dict):
            traffic, issue, capture = tr.get("dram_bytes_per_launch"), tr.get("issue_active_pct"), tr.get("capture")
    roofline = {"kernel": dom, "bound": dk["bound"], "achieved": dk["achieved"],
                "peak": hbm if dk["bound"] == "hbm" else fp32, "unit": dk["unit"], "frac": dk["frac"],
                "traffic": traffic, "issue_active_pct": issue, "ncu_capture": capture,
                "peak_source": (f"{hbm_src} HBM copy (MEASURED_PEAKS.json)" if dk["bound"] == "hbm" else fp32_src),
                "unit_of_work": ("SURVEY.md §8(d): K3 46 flop / K4 120 flop per alpha-passing (blended) pair, "
                                 "K1 12 B per Gaussian + 300 B per visible, K5 600 B per visible (batched K5: "
                                 "DESIGN.md §7)")}

    # kernel launches (all ours, librade.so): per view K1, K2h, 4 depth passes, scan, the tile
    # passes (the first fused with the duplicate generation), ranges, tile order, K3, K4,
    # K5b + K5b64 (batched K5: one of each per round, blockIdx.y = view); per round of views
    # the batched SH kernel (or K5a per view)
    launches_per_view = 1 + 1 + 4 + 1 + tile_passes + 1 + 1 + 1 + 1 + 2
    views_per_rank = args.steps * B
    rounds = args.steps * math.ceil(B / P_)
    launches_total = launches_per_view * views_per_rank + (rounds if args.k5 in ("batched", "split", "set", "split-set") else views_per_rank)
    if args.k5 in ("batched", "set"):  # the round's geometry parts: one K5b64 + one K5b launch per round
        launches_total += 2 * rounds - 2 * views_per_rank
    if args.k1 == "batched":  # one K1 per round instead of one per view
        launches_total += rounds - views_per_rank
    M_avg = tim["n_duplicates"] / max(views_timed, 1)
    vis_avg = tim["n_visible"] / max(views_timed, 1)
    config.update({
        "views_per_step_per_rank": B, "views_timed": total_views,
        "l2": "inputs larger than L2: 354 MB of Gaussian parameters streamed per view (126 MB L2)"
        if n >= 1_000_000 else "small config",
        "M_per_view": M_avg, "visible_per_view": vis_avg, "tiles_per_visible": M_avg / max(vis_avg, 1),
        "culled_per_view": {k: v / max(views_timed, 1) for k, v in tim["n_culled"].items()},
        "pairs_evaluated_per_px_fwd": tim["pairs_evaluated_fwd"] / max(views_timed, 1) / (H * W),
        "pairs_blended_per_px": tim["pairs_blended_fwd"] / max(views_timed, 1) / (H * W),
        # E_issued = K3 warp steps × 64 pixels; E_px / E_issued = the SIMT efficiency
        "pairs_issued_per_px_fwd": tim.get("pairs_issued_fwd", 0) / max(views_timed, 1) / (H * W),
        "simt_efficiency_fwd": tim["pairs_evaluated_fwd"] / max(tim.get("pairs_issued_fwd", 0), 1),
        "ms_per_view_by_kernel": {k: tim["ms"][k] / max(views_timed, 1) for k in tim["ms"]},
        "step_ms": {"median": float(np.median(step_ms)), "mean": float(step_ms.mean()),
                    "p10": float(np.percentile(step_ms, 10)), "p90": float(np.percentile(step_ms, 90)),
                    "per_view_median": float(np.median(step_ms)) / B, "per_view_mean": float(step_ms.mean()) / B,
                    "what": "device time per step (CUDA events on the main stream, this rank), and per view = / B"},
        "views_covered_per_rank": f"{views_covered} of the rank's {len(my_views)} views in the timed steps",
        "parallelism": f"view-parallel dp{ws}",
        "streams": P_, "host_threads": bool(args.host_threads),
        "allreduce": (f"NCCL sum of the {4 * fg.flat.numel() / 2**20:.0f} MB flat gradient buffer once per step, "
                      f"{args.bucket_mb} MB buckets on a side stream" if dist_on else "none (N = 1)"),
    })
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config,
            "roofline": roofline, "kernels": kernels, "gpu_launches": launches_total,
            "clocks": clk, "e2e": e2e}

    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cam = my_views[0]
        t, desc, cores, spent = oracle_frame_time(scene, cam, opt, n_pix=args.cpu_pixels, n_grad=args.cpu_grads,
                                                  seed=0)
        line["cpu_baseline"] = {"value": 1.0 / t, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
    if rank == 0:
        print(json.dumps(line), flush=True)
    for sl in slots:
        sl["view"].close()
    if dist_on:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50, help="timed steps (50 × 4 views = one pass over C3's 200 views)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="rade", choices=["rade", "reference"])
    ap.add_argument("--config", default="C3", choices=["C0", "C1", "C2", "C3", "C4"])
    ap.add_argument("--views-per-step", default="4",
                    help="views per rank per step, or 'epoch' (ceil(views / ranks): one all-reduce per epoch)")
    ap.add_argument("--bucket-mb", type=int, default=64, help="all-reduce bucket size (N > 1)")
    ap.add_argument("--k5", default="set", choices=["set", "batched", "split", "split-set", "per-view"],
                    help="K5 of a round of views in one call: 'set' (default) sets the SH gradient rows in the "
                         "step's first round (RD_K5_SET_SH; only the other gradients are zeroed), 'batched' "
                         "accumulates all; 'split' runs the geometry parts per view; or 'per-view'")
    ap.add_argument("--k1", default="batched", choices=["batched", "per-view"],
                    help="K1 per view on its stream, or one rd_preprocess_views launch per round of views")
    ap.add_argument("--guard-band", type=float, default=None,
                    help="reading S6b guard band (0 = off); default: the config's (C3/C4 0.15, others off)")
    ap.add_argument("--dry-run-gloo", action="store_true",
                    help="CPU-only rehearsal of the distributed step (gloo, fake per-view work): plumbing test")
    ap.add_argument("--n-gaussians", type=int, default=None)
    ap.add_argument("--ref-pixels", type=int, default=32, help="oracle arm: forward pixels sampled per step")
    ap.add_argument("--ref-grads", type=int, default=2, help="oracle arm: Gaussians differentiated per step")
    ap.add_argument("--cpu-pixels", type=int, default=2048, help="cpu_baseline: forward pixels sampled")
    ap.add_argument("--cpu-grads", type=int, default=64, help="cpu_baseline: Gaussians differentiated")
    ap.add_argument("--tile", type=int, default=8, choices=[8, 16, 32], help="blend tile edge (outputs are tile-size independent)")
    ap.add_argument("--distortion", action="store_true", help="NEXT-1: also render L_d and back-propagate it")
    ap.add_argument("--normal-consistency", action="store_true",
                    help="NEXT-2: also compute L_n on the maps and back-propagate it")
    ap.add_argument("--pipeline", type=int, default=0,
                    help="CUDA streams (and host threads) the views are pipelined over; 0 = views per step (max 8)")
    ap.add_argument("--single-host-thread", dest="host_threads", action="store_false",
                    help="issue every view from the main thread (default: one host thread per stream)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--nccl-single", action="store_true",
                    help="at N = 1, run the multi-GPU code path anyway (an NCCL group of one rank)")
    ap.add_argument("--k1-groups", type=int, default=1,
                    help="--k1 batched: the round's views in this many batched K1 launches (1 = one launch)")
    ap.add_argument("--prio", default="none", choices=["none", "views", "views-k5"],
                    help="stream priorities: views = the round's earlier views on higher-priority streams "
                         "(they finish binning first and their K3/K4 fill the others' latency gaps); "
                         "views-k5 = also the K5 stream highest")
    ap.add_argument("--stagger", type=int, default=0,
                    help="view k of a round starts once view k - S is binned (0: all views at once)")
    ap.add_argument("--e2e-mode", default="loss", choices=["loss", "maps"],
                    help="e2e inputs/outputs: GT images in + loss out (default), or cotangent images in + maps out")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 does not meet the timing rules", file=sys.stderr)
    rc = relaunch_if_needed(args)
    if rc is not None:
        return rc
    import scenegen as sg
    info = sg.CONFIGS[args.config]
    config = {"workload": f"{args.config}: {info['name']}", "width": info["width"], "height": info["height"],
              "n_gaussians": args.n_gaussians or info["n"], "sh_degree": 3, "tile": args.tile,
              "depth_distortion": args.distortion,
              "normal_consistency": args.normal_consistency,
              "scene_recipe": "scenegen (DESIGN.md §Input recipe), seed 0 + config index"}
    if args.impl == "reference":
        return run_reference(args, args.config, config)
    if args.dry_run_gloo:
        return run_dry_gloo(args, args.config, config)
    return run_gpu(args, args.config, config)


if __name__ == "__main__":
    sys.exit(main())
