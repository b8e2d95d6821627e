"""Benchmark: hybrid-GS fwd+bwd iters/s (and fwd frames/s) at 1M Gaussians, 1080p.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): synthetic 1M-Gaussian mixed
2D/3D scene, SH degree 3, 1920x1080, seeded generator; one step = forward
render + backward (KG = 1 colour gradient) of one view, inputs resident in HBM.
Under torchrun (N > 1) every rank renders its own view of the replicated scene
(camera sharding, weak scaling) and the per-Gaussian gradient buffer is
all-reduced over NCCL each step -- the multi-view training exchange.

One JSON line on rank 0 (see the keys below).  Timing: W untimed warm-up
steps; K timed steps, each bracketed by CUDA events on the launching stream
with an L2 flush (256 MiB write) between steps outside the events; barrier +
synchronize around the timed region; the max over ranks is reported.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

MEASURED_PEAKS = os.path.join(REPO, "MEASURED_PEAKS.json")
NCU_TAG = "r02"  # profiles/ncu_<tag>_kernels.json: the committed capture the roofline limiter quotes
METRIC = "hybrid-GS frames/s fwd & iters/s fwd+bwd at 1M Gaussians 1080p; 1/2/4/8 B200"
N_SM = 148
FMA_PER_SM_CLK = 128
MUFU_PER_SM_CLK = 16
N_BUCKETS = 4  # gradient all-reduce buckets (parallel.view_batch_grads)

# Algorithmic work per pair (_blend_py.py:17-44, 96-113, 149-240)
FLOP_EVAL_3D = 13       # distance + alpha of a bbox-passing 3D pair
FLOP_EVAL_2D = 34       # ray-splat solve + low-pass + alpha of a 2D pair
FLOP_CONTRIB = 11       # weight, colour, depth, transmittance update
FLOP_BWD_3D = 60        # per contributing pair per KG
FLOP_BWD_2D_RAY = 115
FLOP_BWD_2D_LP = 40


def init_dist(dev):
    """NCCL process group (one process per GPU).  HGS_DIST_BACKEND=gloo runs
    the same multi-rank code path with several ranks on one GPU (a logic
    check on single-GPU boxes; NCCL refuses duplicate devices)."""
    import torch
    import torch.distributed as dist
    backend = os.environ.get("HGS_DIST_BACKEND", "nccl")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if backend == "nccl":
        if torch.cuda.device_count() < world:
            raise SystemExit("bench.py: %d ranks need %d GPUs for NCCL (this box has %d); set "
                             "HGS_DIST_BACKEND=gloo to run the ranks on shared GPUs"
                             % (world, world, torch.cuda.device_count()))
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)


def self_launch(a):
    """``bench.py --gpus N`` without a launcher: re-exec under
    torch.distributed.run with N ranks on this node (127.0.0.1).  Returns the
    launcher's exit code, or None when already inside a launched rank."""
    if a.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
           str(a.gpus), "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def rank_camera(cam, rank):
    """Config 2 under N ranks: rank r renders its own view of the replicated
    scene -- the config-2 camera translated by 0.05 r along x (about 15 px of
    parallax at the scene's median depth; rank 0 = the single-GPU view)."""
    if rank == 0:
        return cam
    from paper_2512_02932_b200.synthetic import synthetic_camera
    w2c = np.array(cam.world_to_camera, dtype=np.float64)
    w2c[0, 3] -= 0.05 * rank
    return synthetic_camera(cam.width, cam.height, w2c)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5],
                    help="BASELINE.json config: 2 (headline, default), 3 (DTU-like + exchange), "
                         "4 (3M Gaussians, full frequency-decoupled training step), "
                         "5 (64-view batch sharded over the GPUs)")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--sh-degree", type=int, default=3)
    ap.add_argument("--kg", type=int, default=1)
    ap.add_argument("--fast", action="store_true", help="HGS_FLAG_FAST (skip f64 re-checks)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-warmup", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=1, help="full-frame CPU baseline steps")
    ap.add_argument("--graph", action="store_true",
                    help="replay fwd+bwd from a CUDA graph (measured: fwd+bwd 3.75 vs 3.67 ms eager, "
                         "fwd 1.69 vs 1.71 ms)")
    return ap.parse_args()


def workload_config(a, n_gpus):
    return {"workload": "synthetic %d-Gaussian mixed 2D/3D scene (50/50), SH deg %d, %dx%d, "
                        "fwd + bwd (KG=%d) per view, one view per GPU per step"
                        % (a.n, a.sh_degree, a.width, a.height, a.kg),
            "n_gaussians": a.n, "width": a.width, "height": a.height, "sh_degree": a.sh_degree,
            "kg": a.kg, "views_per_gpu_per_step": 1,
            "parallelism": "camera-sharded dp%d (a distinct view per rank) + %s all-reduce of the "
                           "gradient buffer in %d buckets overlapped with the chain rule"
                           % (n_gpus, os.environ.get("HGS_DIST_BACKEND", "nccl").upper(), N_BUCKETS)
            if n_gpus > 1 else "single GPU",
            "l2": "flushed between timed steps (256 MiB write); scene (237 MB) > L2 (126 MB)",
            "decisions": "fast (f32 only)" if a.fast else "exact (f64 re-check near thresholds)"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML
    polled every 10 ms from a thread (nvidia-smi -lms 200 as a fallback), so
    even a sub-second timed region yields tens of samples."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index, period_s=0.01):
        self.gpu = gpu_index
        self.period = period_s
        self.sm, self.mx, self.reasons = [], [], set()
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[0].isdigit() else self.gpu
            self.nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx))
            self.t = threading.Thread(target=self._poll_nvml, daemon=True)
        except Exception:
            self.nvml = None
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                     "--format=csv,noheader,nounits", "-lms", "200"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._read_smi, daemon=True)
            except OSError:
                self.proc = None
                return self
        self.t.start()
        return self

    def _poll_nvml(self):
        nv, h = self.nvml
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        while True:
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for nm, b in bits.items():
                    if r & b:
                        self.reasons.add(nm)
            except Exception:
                pass
            if self.stop.wait(self.period):
                return

    def _read_smi(self):
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            if r[1].replace(".", "").isdigit():
                self.sm.append(float(r[1]))
            if r[2].replace(".", "").isdigit():
                self.mx.append(float(r[2]))
            for nm, v in zip(self.NAMES, r[5:9]):
                if v.lower() == "active":
                    self.reasons.add(nm)

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.nvml is not None or self.proc is not None:
            self.t.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml 10 ms" if self.nvml is not None else "nvidia-smi 200 ms"}


# ------------------------------------------------------------ CPU baseline
def _host_threads():
    # all host cores (torchrun sets OMP_NUM_THREADS=1 per rank)
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def cpu_frame_step(scene, cam, st, kg=1, seed=0):
    """One full step of the reference's CPU path on the whole frame (no crop,
    no extrapolation): build_frame + forward blend + backward (blend replay +
    chain rule) on all host cores.  Returns (seconds, fwd seconds, parts)."""
    import oracle
    oracle.set_num_threads(_host_threads())
    rng = np.random.default_rng(seed)
    pg = rng.normal(size=(kg, cam.height, cam.width, 3))
    t0 = time.perf_counter()
    f = oracle.build_frame(scene, cam, st)
    t1 = time.perf_counter()
    oracle.render(scene, cam, st, frame=f)
    t2 = time.perf_counter()
    oracle.backward(scene, cam, st, pg, frame=f)
    t3 = time.perf_counter()
    return t3 - t0, t2 - t0, (t1 - t0, t2 - t1, t3 - t2)


def cpu_baseline(scene, cam, st, kg=1, steps=1):
    """The oracle port (float64 C restatement of the reference CPU path) on all
    host cores, timed on full 1080p frames of the same workload."""
    import oracle
    ts, tf, parts = [], [], None
    for i in range(steps):
        t, f, parts = cpu_frame_step(scene, cam, st, kg, seed=i)
        ts.append(t)
        tf.append(f)
    t_iter, t_fwd = float(np.mean(ts)), float(np.mean(tf))
    return {"value": 1.0 / t_iter, "unit": "iters/s", "cores": oracle.num_threads(),
            "kind": "port", "fwd_frames_per_s": 1.0 / t_fwd,
            "sample": "oracle/hgs_oracle.c (float64, OpenMP, %d threads): %d full %dx%d step(s) on "
                      "all %d Gaussians, measured (no crop, no extrapolation): build_frame %.2fs + "
                      "forward blend %.2fs + backward %.2fs (last step)"
                      % ((oracle.num_threads(), steps, cam.width, cam.height, scene.count) + parts)}


def run_reference(a):
    """--impl reference: the reference's CPU path (the oracle port, all host
    threads) on the same workload, full frames; rank 0 only.  Warm-up is one
    step and the timed steps are capped so the run stays within ~2 minutes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_2512_02932_b200.settings import RenderSettings
    from paper_2512_02932_b200.synthetic import synthetic_scene
    scene, cam = synthetic_scene(a.n, a.width, a.height, a.sh_degree, seed=0)
    st = RenderSettings()
    budget_s = float(os.environ.get("HGS_REF_BUDGET_S", "120"))
    t_w = 0.0
    for i in range(min(a.warmup, 1)):
        t_w = cpu_frame_step(scene, cam, st, a.kg, seed=1000 + i)[0]
    steps = a.steps
    if t_w > 0:
        steps = max(1, min(a.steps, int(budget_s / t_w)))
    ts, tf, parts = [], [], None
    for i in range(steps):
        t, f, parts = cpu_frame_step(scene, cam, st, a.kg, seed=i)
        ts.append(t)
        tf.append(f)
    v = 1.0 / float(np.mean(ts))
    cb = {"value": v, "unit": "iters/s", "cores": oracle.num_threads(), "kind": "port",
          "fwd_frames_per_s": 1.0 / float(np.mean(tf)),
          "sample": "oracle/hgs_oracle.c (float64, OpenMP, %d threads): %d timed full %dx%d "
                    "fwd+bwd steps (+%d warm-up; --steps %d capped to a %.0f s budget), all %d "
                    "Gaussians, measured: build_frame %.2fs + forward blend %.2fs + backward %.2fs "
                    "(last step)" % ((oracle.num_threads(), steps, a.width, a.height, min(a.warmup, 1),
                                     a.steps, budget_s, a.n) + parts)}
    line = {"metric": METRIC, "value": v, "unit": "iters/s", "n_gpus": a.gpus, "steps": steps,
            "warmup": min(a.warmup, 1), "ms_per_step": 1000.0 / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(a, 1), "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- our arm
def run_extra(a):
    """--config 3 / 5 (BASELINE.json configs[2], configs[4]); evidence lines,
    the driver's headline run is config 2."""
    import torch
    import torch.distributed as dist

    from paper_2512_02932_b200 import _lib, exchange, grad, parallel, raster
    from paper_2512_02932_b200.core import DeviceGaussians
    from paper_2512_02932_b200.settings import ExchangeConfig, RenderSettings
    from paper_2512_02932_b200.synthetic import f32_exact, orbit_cameras, synthetic_scene

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        init_dist(dev)
    st = RenderSettings()
    flags = _lib.HGS_FLAG_FAST if a.fast else 0
    if a.config == 3:
        n, W, H = 300_000, 800, 600
        scene, cam = synthetic_scene(n, W, H, 3, seed=0)
        cams, views = [cam], [0]
        workload = ("config 3: synthetic 300k-Gaussian mixed scene, 800x600, SH 3, RGB + depth + "
                    "normal outputs and upstream gradients, Adaptive Type Exchange pass every step")
        unit = "iters/s"
    else:
        n, W, H = a.n, a.width, a.height
        scene, _ = synthetic_scene(n, W, H, 3, seed=0)
        scene.center[:] = f32_exact(scene.center - scene.center.mean(axis=0))
        cams = orbit_cameras(scene, 64, W, H, radius=5.0)
        views = parallel.shard_views(len(cams), rank, world)
        workload = ("config 5: synthetic 1M-Gaussian scene centred at the origin, 64 cameras on a "
                    "circle of radius 5, 1920x1080, fwd + bwd per view, views sharded over %d GPU(s), "
                    "one gradient all-reduce per step" % world)
        unit = "views/s"
    ds = DeviceGaussians.from_host(scene, dev)
    P = 11 + 3 * ds.sh_bases
    if a.config == 3 and world > 1:  # one view per rank: a distinct camera each (camera sharding)
        cams = [rank_camera(cam, rank)]
    gen = torch.Generator(device=dev).manual_seed(99 + rank)
    pg = torch.randn((1, H, W, 3), device=dev, generator=gen)
    dg = torch.randn((1, H, W), device=dev, generator=gen) * 0.1 if a.config == 3 else None
    ng = torch.randn((1, H, W, 3), device=dev, generator=gen) * 0.1 if a.config == 3 else None
    acc = torch.zeros(n * P, dtype=torch.float32, device=dev)
    tbuf = torch.empty(n, dtype=torch.uint8, device=dev)
    scratch = torch.empty(_lib.lib().hgs_backward_scratch_bytes(n, 1), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    xcfg = ExchangeConfig()
    info = {}

    def step():
        # every view's gradient summed by the chain rule itself (HGS_FLAG_ACCUMULATE),
        # the all-reduce bucketed and overlapped with the last view's chain rule
        frame = parallel.view_batch_grads(ds, [cams[v] for v in views], st, lambda j, im: pg, acc,
                                          scratch=scratch, touched=tbuf, flags=flags,
                                          buckets=N_BUCKETS, ext_grads=(dg, ng, None))
        if frame is not None:
            info["K"] = frame.pair_count
        if a.config == 3:
            info["exchange"] = exchange.exchange_pass_device(ds, xcfg)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s_ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    e_ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    with ClockSampler(local) as clocks:
        for i in range(a.steps):
            flush.fill_(i & 0xff)
            s_ev[i].record()
            step()
            e_ev[i].record()
        torch.cuda.synchronize()
    ms = float(np.mean([s_ev[i].elapsed_time(e_ev[i]) for i in range(a.steps)]))
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    per_step = len(cams) if a.config == 5 else 1
    value = per_step * 1000.0 / ms if a.config == 5 else world * 1000.0 / ms
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong" if a.config == 5 else "weak", "vs_baseline": None,
                "dtype": "fp32", "data": "synthetic (seeded generator, SURVEY.md 8d)",
                "config": {"workload": workload, "n_gaussians": n, "width": W, "height": H,
                           "views_per_step": per_step, "l2": "flushed between timed steps"},
                "clocks": clocks.summary(), "last_K_pairs": info.get("K")}
        if a.config == 3 and "exchange" in info:
            rep = info["exchange"]
            line["exchange_last_step"] = {"n_3d_to_2d": rep.n_3d_to_2d, "n_2d_to_3d": rep.n_2d_to_3d,
                                          "n_2d": rep.n_2d, "n_3d": rep.n_3d}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_train(a):
    """--config 4 (BASELINE.json configs[3]): 3M-Gaussian synthetic scene at
    1080p, SH 3; one step = the full frequency-decoupled training step of one
    view: render -> L_color / L_low / L_high and their
    (3, H, W, 3) upstream gradients -> backward with KG = 3 -> per-Gaussian
    gradient surgery (Alg. 1, projection mode) -> Adam -> quaternion
    renormalisation.  Under torchrun every rank trains on its own view and the
    combined gradient is all-reduced before the (replicated) Adam step."""
    import torch
    import torch.distributed as dist

    from paper_2512_02932_b200 import freq, grad, optim, parallel, raster
    from paper_2512_02932_b200.core import DeviceGaussians
    from paper_2512_02932_b200.settings import RenderSettings
    from paper_2512_02932_b200.synthetic import synthetic_scene

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        init_dist(dev)
    n = 3_000_000 if a.n == 1_000_000 else a.n
    W, H = a.width, a.height
    scene, cam = synthetic_scene(n, W, H, 3, seed=0)
    cam = rank_camera(cam, rank)  # each rank trains on its own view
    st = RenderSettings()
    ds = DeviceGaussians.from_host(scene, dev)
    # target image: render of an independent scene of the same statistics
    tscene, _ = synthetic_scene(n, W, H, 3, seed=100 + rank)
    gt_imgs, _ = raster.rasterize(DeviceGaussians.from_host(tscene, dev), cam, st)
    gt = gt_imgs["color"].clone()
    del tscene, gt_imgs
    w = freq.LossWeights()
    opt = optim.Adam(ds)
    P = 11 + 3 * ds.sh_bases
    comb = torch.empty(n * P, dtype=torch.float32, device=dev) if world > 1 else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def step(evs=None):
        if world == 1:
            return optim.train_step(ds, cam, gt, opt, w, st, events=evs)
        if evs:
            evs[0].record()
        imgs, frame = raster.rasterize(ds, cam, st)
        if evs:
            evs[1].record()
        losses, stack = freq.image_losses(imgs["color"], gt, w)
        if evs:
            evs[2].record()
        g, _ = grad.backward_device(frame, stack)
        if evs:
            evs[3].record()
        nc = freq.combine_gradients_device(g[0], g[1], g[2], ds.type_spec, w.mode, out=comb)[1]
        parallel.allreduce_grads(comb)
        opt.step(comb)
        return optim.TrainStepResult(losses, nc, frame.pair_count, imgs["color"])

    for _ in range(a.warmup):
        res = step()
    torch.cuda.synchronize()
    l0 = res.losses.cpu().tolist()
    if world > 1:
        dist.barrier()
    K = a.steps
    s_ev = [ev() for _ in range(K)]
    e_ev = [ev() for _ in range(K)]
    st_ev = [[ev() for _ in range(4)] for _ in range(K)]
    with ClockSampler(local) as clocks:
        for i in range(K):
            flush.fill_(i & 0xff)
            s_ev[i].record()
            res = step(st_ev[i])
            e_ev[i].record()
        torch.cuda.synchronize()
    ms = float(np.mean([s_ev[i].elapsed_time(e_ev[i]) for i in range(K)]))
    names = ["render", "losses(L1+SSIM+DWT, KG=3 stack)", "backward(KG=3)"]
    stages = {nm: float(np.mean([st_ev[i][j].elapsed_time(st_ev[i][j + 1]) for i in range(K)]))
              for j, nm in enumerate(names)}
    stages["surgery+adam(+allreduce)"] = float(np.mean([st_ev[i][3].elapsed_time(e_ev[i])
                                                       for i in range(K)]))
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    peaks = json.load(open(MEASURED_PEAKS)) if os.path.exists(MEASURED_PEAKS) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    # HBM roofline of the two new HBM-bound stages (algorithmic bytes)
    loss_bytes = H * W * 3 * 52 + 0
    opt_bytes = n * 4 * P * (6 + 3) if world == 1 else n * 4 * P * (1 + 3 + 3)
    stage_roofs = {
        "losses(L1+SSIM+DWT, KG=3 stack)": {"GB/s": loss_bytes / stages[names[1]] / 1e6,
                                            "hbm_frac": loss_bytes / stages[names[1]] / 1e6
                                            / hbm_peak},
        "surgery+adam(+allreduce)": {"GB/s": opt_bytes / stages["surgery+adam(+allreduce)"] / 1e6,
                                     "hbm_frac": opt_bytes / stages["surgery+adam(+allreduce)"]
                                     / 1e6 / hbm_peak}}
    if rank == 0:
        l1 = res.losses.cpu().tolist()
        line = {"metric": METRIC, "value": world * 1000.0 / ms, "unit": "iters/s", "n_gpus": world,
                "steps": K, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
                "data": "synthetic (seeded generator, SURVEY.md 8d); target = render of an "
                        "independent synthetic scene",
                "config": {"workload": "config 4: synthetic %d-Gaussian scene, %dx%d, SH 3, full "
                                       "frequency-decoupled training step per view (render, "
                                       "L_color/L_low/L_high, backward KG=3, gradient surgery "
                                       "(projection), Adam, quaternion renormalisation)"
                                       % (n, W, H),
                           "n_gaussians": n, "width": W, "height": H, "views_per_gpu_per_step": 1,
                           "parallelism": "dp%d (combined gradient all-reduced)" % world
                           if world > 1 else "single GPU",
                           "l2": "flushed between timed steps (256 MiB write)"},
                "stages_ms": stages, "stage_rooflines": stage_roofs, "clocks": clocks.summary(),
                "K_pairs": res.pair_count,
                "loss_first_warmup_step": l0, "loss_last_step": l1,
                "n_conflicts_last_step": int(res.n_conflicts.item())}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    rc = self_launch(a)
    if rc is not None:
        sys.exit(rc)
    if a.config == 4:
        run_train(a)
        return
    if a.config in (3, 5):
        run_extra(a)
        return
    import torch
    import torch.distributed as dist

    from paper_2512_02932_b200 import _lib, grad, parallel, raster
    from paper_2512_02932_b200.core import DeviceGaussians
    from paper_2512_02932_b200.settings import RenderSettings
    from paper_2512_02932_b200.synthetic import synthetic_scene

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        init_dist(dev)
        if a.kg != 1:
            raise SystemExit("bench.py: the multi-rank step sums KG = 1 view gradients")

    scene, cam0 = synthetic_scene(a.n, a.width, a.height, a.sh_degree, seed=0)
    cam = rank_camera(cam0, rank)  # distinct view per rank (camera sharding)
    st = RenderSettings()
    ds = DeviceGaussians.from_host(scene, dev)
    flags = _lib.HGS_FLAG_FAST if a.fast else 0
    H, W = a.height, a.width
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    pg = torch.randn((a.kg, H, W, 3), device=dev, generator=g)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    n, P = ds.count, 11 + 3 * ds.sh_bases
    grads_buf = torch.empty((a.kg, n * P), dtype=torch.float32, device=dev)
    touched_buf = torch.empty(n, dtype=torch.uint8, device=dev)
    scratch = torch.empty(_lib.lib().hgs_backward_scratch_bytes(n, a.kg), dtype=torch.uint8,
                          device=dev)
    imgs = dict(color=torch.empty((H, W, 3), device=dev), depth=torch.empty((H, W), device=dev),
                transmittance=torch.empty((H, W), device=dev), alpha=torch.empty((H, W), device=dev),
                normal=torch.empty((H, W, 3), device=dev))

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def step(fe=None, be=None):
        if world > 1:  # the multi-view gradient exchange, bucketed and overlapped
            return parallel.view_batch_grads(ds, [cam], st, lambda j, im: pg, grads_buf[0],
                                             scratch=scratch, touched=touched_buf, flags=flags,
                                             buckets=N_BUCKETS, events=be, fwd_events=fe,
                                             outputs=imgs)
        # no host round trip inside a step (HGS_FLAG_ASYNC); the frames'
        # statuses are checked after the timed region
        _, frame = raster.rasterize(ds, cam, st, flags, outputs=imgs, events=fe, async_=True,
                                    frame_buf=fbuf)
        grad.backward_device(frame, pg, grads_out=grads_buf, touched_out=touched_buf, events=be,
                             scratch=scratch)
        return frame

    def fwd_only(fe=None):
        _, frame = raster.rasterize(ds, cam, st, flags, outputs=imgs, events=fe, async_=True,
                                    frame_buf=fbuf)
        return frame

    # ---- counting pass (outside timing): algorithmic work per launch
    _, cframe = raster.rasterize(ds, cam, st, flags | _lib.HGS_FLAG_COUNT, outputs=imgs)
    grad.backward_device(cframe, pg, grads_out=grads_buf, touched_out=touched_buf,
                         flags=flags | _lib.HGS_FLAG_COUNT, scratch=scratch)
    stats = _lib.frame_stats(cframe).astype(np.int64)
    M, K = cframe.count, cframe.pair_count
    n_depth_passes, n_tile_passes = int(cframe.info.internal[2]), int(cframe.info.internal[3])
    del cframe
    # one frame buffer for every timed frame, sized from the counting pass
    fbuf = torch.empty(raster.frame_bytes(n, W, H), dtype=torch.uint8, device=dev)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()

    # --graph (single GPU): a step is replayed from a CUDA graph (a frame is
    # enqueued with no host round trip, so forward + backward capture as one
    # graph; the L2 flush stays outside it), the stage split from the same
    # steps run eagerly with the library's stage events.  Eager launches are
    # the default: they measured faster for forward + backward.
    use_graph = world == 1 and a.graph
    g_step = g_fwd = None
    if use_graph:
        g_step, g_fwd = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_step):
            step()
        with torch.cuda.graph(g_fwd):
            graph_frame = fwd_only()
        g_step.replay()
        g_fwd.replay()
        torch.cuda.synchronize()

    # ---- timed fwd+bwd steps
    K_ = a.steps
    s_ev = [ev() for _ in range(K_)]
    e_ev = [ev() for _ in range(K_)]
    f_ev = [[ev() for _ in range(5)] for _ in range(K_)]
    b_ev = [[ev() for _ in range(3)] for _ in range(K_)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # the timed steps carry only the backward's stage events (the dominant
    # kernel's duration for the roofline is taken inside the timed region);
    # the forward's stage events -- a library event between two kernels also
    # breaks their programmatic dependent launch -- come from a separate,
    # untimed pass of K eager steps below
    with ClockSampler(local) as clocks:
        for i in range(K_):
            flush.fill_(i & 0xff)
            s_ev[i].record()
            if use_graph:
                g_step.replay()
            else:
                step(None, b_ev[i])
            e_ev[i].record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # fwd-only frames/s
        fs = [ev() for _ in range(K_)]
        fe = [ev() for _ in range(K_)]
        for i in range(K_):
            flush.fill_(i & 0xff)
            fs[i].record()
            if use_graph:
                g_fwd.replay()
            else:
                last_frame = fwd_only()
            fe[i].record()
        torch.cuda.synchronize()
    if use_graph:
        last_frame = graph_frame
    b_ev2 = [[ev() for _ in range(3)] for _ in range(K_)]
    for i in range(K_):  # the forward's stage split, eagerly (library stage events), untimed
        flush.fill_(i & 0xff)
        step(f_ev[i], b_ev2[i] if not use_graph else b_ev[i])
    torch.cuda.synchronize()
    last_frame.sync()  # raises if a timed frame overflowed its pair capacity (none did: same K every step)
    step_ms = float(np.mean([s_ev[i].elapsed_time(e_ev[i]) for i in range(K_)]))
    fwd_ms = float(np.mean([fs[i].elapsed_time(fe[i]) for i in range(K_)]))
    stage_names = ["depth_keys+sort||preprocess_f64", "scan", "binning(dup+tile sort+ranges)",
                   "composite_fwd"]
    stages = {}
    for j, nm in enumerate(stage_names):
        stages[nm] = float(np.mean([f_ev[i][j].elapsed_time(f_ev[i][j + 1]) for i in range(K_)]))
    stages["composite_bwd"] = float(np.mean([b_ev[i][0].elapsed_time(b_ev[i][1]) for i in range(K_)]))
    stages["chain_rule(+touched)"] = float(np.mean([b_ev[i][1].elapsed_time(b_ev[i][2])
                                                   for i in range(K_)]))
    if world > 1:
        t = torch.tensor([step_ms, fwd_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms, fwd_ms = float(t[0]), float(t[1])

    clk = clocks.summary()
    sm_mhz = clk["sm_mhz"] or 1965.0
    fp32_peak = N_SM * FMA_PER_SM_CLK * 2 * sm_mhz * 1e6 / 1e12
    mufu_peak = N_SM * MUFU_PER_SM_CLK * sm_mhz * 1e6 / 1e12

    # ---- roofline of the dominant kernel
    ev3, ev2, c3, c2 = (int(x) for x in stats[2:6])
    b3, br, bl, bev = (int(x) for x in stats[6:10])
    dom = max(stages, key=stages.get)
    flops = {
        "composite_fwd": FLOP_EVAL_3D * ev3 + FLOP_EVAL_2D * ev2 + FLOP_CONTRIB * (c3 + c2),
        "composite_bwd": (FLOP_EVAL_3D * ev3 + FLOP_EVAL_2D * ev2) * bev / max(ev3 + ev2, 1)
        + a.kg * (FLOP_BWD_3D * b3 + FLOP_BWD_2D_RAY * br + FLOP_BWD_2D_LP * bl),
    }
    mufu = {"composite_fwd": ev3 + 2 * ev2, "composite_bwd": bev + 2 * (b3 + br + bl)}
    hbm_bytes = {
        # depth keys + sort passes + rank scatter, and the preprocess beside them
        "depth_keys+sort||preprocess_f64": a.n * (40 + 2) + a.n * 12 * 2 * n_depth_passes + a.n * 12
        + M * (237 + 96 + 96 + 32 + 8 + 4),
        "scan": M * (8 + 8),
        "binning(dup+tile sort+ranges)": M * 104 + K * (8 + 16 * n_tile_passes + 4),
        "chain_rule(+touched)": a.n * (4 * (11 + 3 * ds.sh_bases) + 1 + 64 * a.kg
                                       + 4 * P * a.kg),
    }
    peaks = json.load(open(MEASURED_PEAKS)) if os.path.exists(MEASURED_PEAKS) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    t_dom = stages[dom] * 1e-3
    if dom in flops:
        ach = flops[dom] / t_dom / 1e12
        roof = {"kernel": dom, "bound": "fp32", "achieved": ach, "peak": fp32_peak,
                "unit": "TFLOP/s", "frac": ach / fp32_peak,
                "mufu_frac": mufu[dom] / t_dom / 1e12 / mufu_peak,
                "peak_source": "148 SM x 128 FFMA/clk x 2 x median SM clock under load "
                               "(%.0f MHz, nvidia-smi during the timed region)" % sm_mhz,
                "work": "%d 3D + %d 2D bbox-passing pairs, %d contributing (fwd); bwd contributing "
                        "3D %d, 2D-ray %d, 2D-lowpass %d" % (ev3, ev2, c3 + c2, b3, br, bl)}
    else:
        ach = hbm_bytes[dom] / t_dom / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                "frac": ach / hbm_peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    # the limiter of the compositors is the SM issue rate, not a pipe peak:
    # quote the committed ncu capture of the same kernel (profiles/)
    ncu_file = os.path.join(REPO, "profiles", "ncu_%s_kernels.json" % NCU_TAG)
    # the instantiation this run launched (template <NAIVE, COUNT, PF> / <KG, EXT, DET, QP>)
    kname = {"composite_fwd": "k_composite_fwd<0, 0, 0, %d>" % (0 if a.fast else 1),
             "composite_bwd": "k_composite_bwd_c<%d, 0, 0, 4, 0>" % min(a.kg, 4)}.get(dom)
    roof["ncu_kernel"] = kname
    roof["traffic"] = None
    if kname and os.path.exists(ncu_file):
        cands = [kd for kd in json.load(open(ncu_file)) if kd.get("kernel") == kname]
        cands.sort(key=lambda kd: kd.get("config") != "c2")  # this workload's capture first
        if cands:
            kd = cands[0]
            roof["limiter"] = ("SM instruction issue (ncu, profiles/ncu_%s_kernels.json, %s capture: issue "
                               % (NCU_TAG, kd.get("config")) +
                               "active %.0f%%, FP32 pipe %.0f%%, DRAM %.0f%%, %.1f of 32 lanes active)"
                               % (kd.get("issue_active_pct", 0), kd.get("fma_pipe_pct", 0),
                                  kd.get("dram_pct", 0), kd.get("thread_inst_per_inst", 0)))
            # dram__bytes_read.sum + dram__bytes_write.sum of that kernel, one launch
            roof["traffic"] = int((kd.get("dram_read_MB", 0) + kd.get("dram_write_MB", 0)) * 1e6)
            roof["traffic_config"] = kd.get("config")
    stage_roofs = {}
    for nm, t_ms in stages.items():
        if nm in flops:
            stage_roofs[nm] = {"ms": t_ms, "TFLOP/s": flops[nm] / (t_ms * 1e-3) / 1e12,
                               "fp32_frac": flops[nm] / (t_ms * 1e-3) / 1e12 / fp32_peak}
        elif nm in hbm_bytes:
            gbs = hbm_bytes[nm] / (t_ms * 1e-3) / 1e9
            stage_roofs[nm] = {"ms": t_ms, "GB/s": gbs, "hbm_frac": gbs / hbm_peak}

    # init_state, depth_keys, sort_plan, 8 depth passes (the constant digits' exit at once),
    # preprocess, tile_counts, rank_scatter, scan_counts, duplicate, radix_offsets, <tile passes>,
    # tile_ranges, composite_fwd, fixup_fwd (the launch list in profiles/launches_r02.csv)
    launches_fwd = 20 + n_tile_passes
    # init_bwd + (composite_bwd + fixup_bwd + chain_rule) per chunk of <= 4 gradients; under
    # N ranks the chain rule runs in N_BUCKETS Gaussian ranges (overlapped all-reduce)
    launches_bwd = 1 + 3 * ((a.kg + 3) // 4) + ((N_BUCKETS - 1) if world > 1 else 0)
    value = world * 1000.0 / step_ms

    # ---- e2e through the public API with host buffers (rank-local)
    e2e = None
    if not a.no_e2e:
        from paper_2512_02932_b200.core import GaussianSet
        host_scene = GaussianSet(scene.center, scene.log_scale, scene.rotation, scene.opacity_logit,
                                 scene.sh_coeffs, scene.type_spec)
        pg_host = pg[0].double().cpu().numpy()
        # the geometry crosses PCIe as float64 (the exact-decision inputs), SH
        # coefficients and the pixel gradient as float32 (converted on the host
        # cores into pinned staging, _hostio.py); uint8 type mask
        h2d = (8 * (host_scene.center.size + host_scene.log_scale.size + host_scene.rotation.size
                    + host_scene.opacity_logit.size)
               + 4 * (host_scene.sh_coeffs.size + pg_host.size) + host_scene.type_spec.size)
        ts = []
        for i in range(a.e2e_warmup + a.e2e_steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = raster.render(host_scene, cam, st, fast=a.fast)
            gr, touched = grad.backward(host_scene, cam, out, pg_host)
            torch.cuda.synchronize()
            if i >= a.e2e_warmup:
                ts.append(time.perf_counter() - t0)
        # the reference's outputs: colour, depth, transmittance, ParamGrads, touched
        # (the extension images alpha / normal download on first access)
        d2h = (4 * (out.color.size + out.depth.size + out.transmittance.size + gr.flat().size)
               + touched.size)
        tt = float(np.mean(ts))
        print("e2e step ms: %s" % " ".join("%.1f" % (1e3 * x) for x in ts), file=sys.stderr)
        if world > 1:
            t = torch.tensor([tt], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tt = float(t[0])
        e2e = {"value": world / tt, "unit": "iters/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "path": "raster.render(GaussianSet float64 numpy) + grad.backward(numpy pixel_grad)"
                       " -> numpy float64 colour / depth / transmittance and ParamGrads (the reference's outputs; the extension images download on first access) (geometry float64, SH / images / gradients float32 over PCIe via pinned staging; float64 <-> float32 conversions on all host cores with streaming stores); wall clock with device syncs"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(scene, cam, st, a.kg, a.cpu_steps)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": step_ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
                "data": "synthetic (seeded generator, SURVEY.md 8d)",
                "config": dict(workload_config(a, world),
                               launch="CUDA graph replay of forward + backward (stage split from the same "
                                      "steps run eagerly)" if use_graph else "eager launches"),
                "fwd_frames_per_s": world * 1000.0 / fwd_ms, "fwd_ms": fwd_ms,
                "stages_ms": stages, "stage_rooflines": stage_roofs, "roofline": roof,
                "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
                "gpu_launches": (launches_fwd + launches_bwd) * a.steps,
                "frame": {"M": M, "K_pairs": K, "depth_sort_passes": n_depth_passes,
                          "f64_rechecks": int(stats[0]), "f64_T_replays": int(stats[1]),
                          "fwd_pairs_evaluated": ev3 + ev2, "fwd_pairs_contributing": c3 + c2}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
