"""Benchmark: decoded+augmented images/s at 224 through the GPU loader.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2|cfg1|cfg4] [--batch B]

Workload (BASELINE.json configs[1], "cfg2"): synthetic 256x256 q95 JPEGs,
crop-decode + RandomResizedCrop(0.08,1)->224 + flip + normalize -> bf16
NCHW, plus MAE-B/16 masking ratio 0.75 (mask ids, ids_keep, ids_restore),
batch 256 per GPU.  A step = one batch through Loader.enqueue (the public
API).  Inputs: an 8192-image pool (~235 MB of compressed bytes, > the 126 MB
L2) resident in HBM, visited in permutation order, so consecutive steps never
hit L2-resident inputs.

`value`  : device-timed whole-job images/s (inputs resident in HBM).
`e2e`    : same metric through Loader.epoch() with host-staged payloads
           (pinned H2D of each batch's JPEG bytes + D2H of per-image status
           inside the timed region).
`roofline`: k_decode (dominant kernel) algorithmic bytes / measured launch
           time (CUDA events around each launch, ESSL_OPT_PROFILE) vs the
           measured HBM copy peak.
`cpu_baseline`: the C oracle (oracle/essl_oracle.c, a port of the reference
           algorithm) on all host cores over a bounded sample.
--impl reference: that CPU implementation as the timed arm.

N>1 (torchrun): one process per GPU, each rank decodes its own DDP shard
(perm[r::world]) -- no collective on the data path; the timing is the max over
ranks (one all_reduce after the timed region).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decoded+augmented images/s at 224 (1/2/4/8 B200) vs host-CPU ref; HBM roofline %"
WORKLOADS = {
    "cfg2": dict(side=256, quality=95, scale=(0.08, 1.0), batch=256, res=224, mask=0.75,
                 desc="256 synthetic 256px q95 JPEGs per batch, crop-decode + RRC(0.08,1)->224 "
                      "+ flip + normalize (bf16 NCHW) + MAE-B/16 mask 0.75 "
                      "(mask/ids_keep/ids_restore)"),
    "cfg1": dict(side=256, quality=95, scale=(0.08, 1.0), batch=256, res=224, mask=0.0,
                 desc="256 synthetic 256px q95 JPEGs per batch, crop-decode + RRC(0.08,1)->224 "
                      "+ flip + normalize (bf16 NCHW)"),
    "cfg4": dict(side=512, quality=90, scale=(0.2, 1.0), batch=1024, res=224, mask=0.0, group=1,
                 desc="1024 synthetic 512px q90 JPEGs per batch, RRC(0.2,1)->224 + flip + "
                      "normalize (bf16 NCHW)"),
    # progressive resolution (schedule.py custom scheme): the
    # timed steps are split evenly over the stages, Loader.retarget between them
    "cfg3": dict(side=256, quality=95, scale=(0.08, 1.0), batch=256, res=224, mask=0.75,
                 schedule=(112, 160, 192, 224),
                 desc="256 synthetic 256px q95 JPEGs per batch, progressive RRC(0.08,1) "
                      "112->160->192->224 (equal steps per stage) + flip + normalize (bf16 "
                      "NCHW) + MAE-B/16 mask 0.75"),
    # epoch-scale stream: 1,281,167 records aliasing a pool
    # of distinct cfg1-style payloads, DDP-sharded perm[r::world]
    "cfg5": dict(side=256, quality=95, scale=(0.08, 1.0), batch=256, res=224, mask=0.75,
                 records=1_281_167,
                 desc="1,281,167-record container (ImageNet-1k size) aliasing the pool of "
                      "256px q95 JPEGs, DDP-sharded epoch stream, batch 256 per GPU, "
                      "RRC(0.08,1)->224 + flip + normalize (bf16 NCHW) + MAE-B/16 mask 0.75"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "src": "fallback"}


def config_dict(args, wl: dict, records: int, mean_payload: float) -> dict:
    """The workload description both arms print (identical keys and values)."""
    return {"workload": f"{args.workload}: {wl['desc']}", "batch": wl["batch"],
            "res": list(wl["schedule"]) if wl.get("schedule") else wl["res"],
            "mask_ratio": wl["mask"], "aug": wl.get("aug", "simple"), "pool_images": args.pool,
            "records": records, "mean_payload_bytes": mean_payload,
            "l2": f"inputs > L2: {args.pool}-image pool (~{args.pool * mean_payload / 1e6:.0f} MB of "
                  "JPEG bytes, 126 MB L2) visited in permutation order; outputs: a reused ring of "
                  "16 output buffers per loader (each written once per 16 steps)",
            "parallelism": "ddp per GPU (rank shards perm[r::world], no collective on the path)",
            "launch_group": getattr(args, "group", 1)}


def dataset_dir(rank: int, ws: int) -> Path:
    """One synthetic dataset per job: under torchrun every rank opens the
    file rank 0 wrote (the other ranks wait on a barrier)."""
    d = Path(tempfile.gettempdir()) / f"essl_bench_{os.environ.get('TORCHELASTIC_RUN_ID', os.getpid())}"
    if ws == 1:
        d = Path(tempfile.mkdtemp(prefix="essl_bench_"))
    d.mkdir(parents=True, exist_ok=True)
    return d


def make_dataset(wl: dict, pool: int, out_dir: Path, seed: int = 1) -> Path:
    from paper_2404_00509_b200 import build_synthetic
    rec = wl.get("records")
    rst = wl.get("restart", 0)
    path = out_dir / f"pool_{wl['side']}_{wl['quality']}_{pool}_{rec or pool}_r{rst}.essl"
    if not path.exists():
        t = time.perf_counter()
        info = build_synthetic(path, pool, wl["side"], wl["quality"], classes=1000, seed=seed,
                               n_records=rec, restart_interval=rst)
        log(f"[bench] built {pool} images ({info['mean_payload']:.0f} B mean) in "
            f"{time.perf_counter() - t:.1f}s")
    return path


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None
        self.marks = []

    def mark(self) -> None:
        """Bracket the timed region (wall clock, matched to sample timestamps)."""
        self.marks.append(time.time())

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self) -> dict:
        import datetime
        rows = []
        try:
            for line in Path(self.path).read_text().splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 10:
                    try:
                        ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                    except ValueError:
                        ts = None
                    rows.append((ts, parts[1:]))
        except OSError:
            pass
        finally:
            if self.path:
                Path(self.path).unlink(missing_ok=True)
        if len(self.marks) >= 2 and rows:
            a, b = self.marks[0], self.marks[-1]
            inside = [r for t, r in rows if t is not None and a - 0.05 <= t <= b + 0.05]
            if not inside:  # timed region shorter than the sampling period: nearest samples
                near = sorted(rows, key=lambda x: abs((x[0] or 0) - (a + b) / 2))[:2]
                inside = [r for _, r in near]
            sel = inside
        else:
            sel = [r for _, r in rows]
        if not sel:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in sel if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in sel if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in sel for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(sel)}


def cpu_oracle_rate(path: Path, wl: dict, seconds: float, seed_epoch=(0, 0)) -> dict:
    """Bounded-sample throughput of the C oracle on all host threads."""
    from oracle import oracle as O
    from paper_2404_00509_b200.container import open_container
    O.build()
    nthreads = os.cpu_count() or 1
    with open_container(path) as h:
        perm = np.random.default_rng(0).permutation(len(h))
        B = wl["batch"]
        pix = np.empty((B, 3, wl["res"], wl["res"]), np.float32)
        done, t0, i = 0, time.perf_counter(), 0
        while True:
            idx = perm[(i * B) % len(h):(i * B) % len(h) + B]
            _, _, _, st = O.loader_batch(h.bytes, h.records, idx, seed_epoch[0], seed_epoch[1],
                                         wl["res"], scale=wl["scale"], mask_ratio=wl["mask"],
                                         aug=wl.get("aug", "simple"),
                                         nthreads=nthreads, pixels=pix[:len(idx)])
            assert (st == 0).all()
            done += len(idx)
            i += 1
            el = time.perf_counter() - t0
            if el >= seconds:
                break
    return {"value": done / el, "unit": "images/s", "cores": nthreads, "kind": "port",
            "sample": f"{done} images ({i} batches of {B}) of the same workload, "
                      f"{el:.1f}s wall, C oracle with {nthreads} threads"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def reference_loader_rates(path: Path, wl: dict, args) -> dict:
    """The unmodified reference cropload.pipeline.Loader (baseline/_ref) on
    this host's cores over the same container: workers = all cores (the
    primary CPU baseline of BASELINE.md section 3), workers = 1, and one
    process per core (upper bound); tools/ref_loader_rate.py, bounded samples."""
    out = {}
    for mode in ("threads", "single", "procs"):
        cmd = [sys.executable, str(ROOT / "tools" / "ref_loader_rate.py"), "--data", str(path),
               "--batch", str(wl["batch"]), "--res", str(wl["res"]), "--scale", str(wl["scale"][0]),
               str(wl["scale"][1]), "--mask", str(wl["mask"]), "--seconds",
               str(args.ref_loader_seconds), "--mode", mode]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
            out[mode] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as e:  # reported, never fatal: the port is the timed arm
            out[mode] = {"unavailable": f"{type(e).__name__}: {e}"[:200]}
    return out


def run_reference(args, wl):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    data_dir = Path(tempfile.mkdtemp(prefix="essl_bench_"))
    path = make_dataset(wl, args.pool, data_dir)
    from oracle import oracle as O
    from paper_2404_00509_b200.container import open_container
    O.build()
    nthreads = os.cpu_count() or 1
    with open_container(path) as h:
        perm = np.random.default_rng(0).permutation(len(h))
        B = wl["batch"]
        pix = np.empty((B, 3, wl["res"], wl["res"]), np.float32)

        def step(i):
            idx = perm[(i * B) % len(h):(i * B) % len(h) + B]
            _, _, _, st = O.loader_batch(h.bytes, h.records, idx, 0, 0, wl["res"],
                                         scale=wl["scale"], mask_ratio=wl["mask"],
                                         aug=wl.get("aug", "simple"),
                                         nthreads=nthreads, pixels=pix[:len(idx)])
            assert (st == 0).all()
            return len(idx)

        for i in range(args.warmup):
            step(i)
        t0 = time.perf_counter()
        n = sum(step(args.warmup + i) for i in range(args.steps))
        el = time.perf_counter() - t0
        records, mean_payload = len(h), float(np.mean(h.records["payload_length"]))
    v = n / el
    ref_loader = reference_loader_rates(path, wl, args) if args.ref_loader_seconds > 0 else None
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "images/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32", "out_dtype": "f32", "data": "synthetic",
            "config": config_dict(args, wl, records, mean_payload),
            "reference_loader": ref_loader,
            "cpu_baseline": {"value": v, "unit": "images/s", "cores": nthreads, "kind": "port",
                             "sample": f"{args.steps} timed batches of {wl['batch']} after "
                                       f"{args.warmup} warm-up, C oracle (port of the reference "
                                       f"algorithm) on {nthreads} threads"},
            "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_gpu(args, wl):
    import torch
    import torch.distributed as dist

    import paper_2404_00509_b200 as E
    from paper_2404_00509_b200 import _native as N
    from paper_2404_00509_b200.ddp import rank_shard

    ws, rank, local = dist_env()
    if ws > 1:
        # ESSL_BENCH_BACKEND=gloo: functional check of the multi-rank path with
        # ranks sharing GPUs (device = local rank mod device count); the data
        # path has no collective either way, only the reporting reduction
        dist.init_process_group(os.environ.get("ESSL_BENCH_BACKEND", "nccl"))
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    data_dir = dataset_dir(rank, ws)
    if rank == 0:
        path = make_dataset(wl, args.pool, data_dir)
    if ws > 1:
        dist.barrier()  # rank 0 has written the dataset; the others open the same file
        path = make_dataset(wl, args.pool, data_dir)  # (exists: no rebuild)
    B, res = wl["batch"], wl["res"]
    cfg = E.LoaderConfig(data=str(path), batch_size=B, res=res, scale=wl["scale"],
                         mask_ratio=wl["mask"], aug=wl.get("aug", "simple"),
                         out_dtype="bfloat16", device=str(dev),
                         rank=rank, world_size=ws, resident=True, prefetch=args.streams,
                         streams=args.streams, reuse_outputs=True, group=args.group)
    loader = E.Loader(cfg)

    def apply_options(ld):  # analysis knobs (library defaults unless given)
        for opt, v, on in ((N.ESSL_OPT_SEQ_BITS, args.seq_bits, args.seq_bits > 0),
                           (N.ESSL_OPT_WARMUP_BITS, args.warm_bits, args.warm_bits >= 0),
                           (N.ESSL_OPT_CHECKPOINT_BITS, args.ck_bits, args.ck_bits > 0),
                           (N.ESSL_OPT_STAGE_BYTES, args.stage_bytes, args.stage_bytes >= 0),
                           (N.ESSL_OPT_RESIZE_COLS, args.resize_cols, args.resize_cols > 0),
                           (N.ESSL_OPT_RESIZE_BAND, args.resize_band, args.resize_band > 0),
                           (N.ESSL_OPT_EARLY_EXIT, args.early_exit, args.early_exit >= 0)):
            if on:
                ld.set_option(opt, v)

    apply_options(loader)
    handle = loader.handle
    perm_epochs = {}
    if args.epoch:  # one full epoch of this rank's shard (whole batches)
        args.steps = max(1, len(handle) // ws // B)

    def batch_indices(i):
        per_epoch = len(handle) // ws // B
        e, j = divmod(i, max(per_epoch, 1))
        if e not in perm_epochs:
            perm_epochs[e] = rank_shard(cfg.seed, e, len(handle), rank, ws)
        return e, perm_epochs[e][j * B:(j + 1) * B]

    stream = torch.cuda.current_stream(dev)
    # The clock sampler starts before the warm-up so that nvidia-smi's own
    # start-up is not inside the timed region; it runs through it.
    clk = Clocks(local).__enter__()
    # ---- warm-up: the same pipelined issue pattern as the timed loop, so the
    # caching allocator and every stream's context reach steady state
    pend = []
    ring_depth = 2 * max(cfg.prefetch, cfg.streams) + 2  # pipeline.py _HostRing slots
    n_warm = max(args.warmup, args.streams * (ring_depth + 1))
    sched = wl.get("schedule")
    G = args.group

    def issue(i, steps, stage_of, g):
        """Batch i (+ up to g-1 following ones of the same epoch and stage) in
        one launch set; returns (pendings, batches issued)."""
        e, idx = batch_indices(i)
        parts = [idx]
        while len(parts) < g and i + len(parts) < steps:
            e2, idx2 = batch_indices(i + len(parts))
            if e2 != e or stage_of(i + len(parts)) != stage_of(i):
                break
            parts.append(idx2)
        if len(parts) == 1:
            return [loader.enqueue(e, idx)], 1
        return loader.enqueue_group(e, parts), len(parts)

    i = 0
    while i < n_warm:
        if sched:  # every stage's output ring allocated before the timed region
            loader.retarget(res=sched[i * len(sched) // n_warm])
        ps, k = issue(i, n_warm, lambda j: j * len(sched) // n_warm if sched else 0, G)
        pend.extend(ps)
        i += k
        while len(pend) > 2 * args.streams * G:
            loader.finish(pend.pop(0))
    for p in pend:
        loader.finish(p)
    torch.cuda.synchronize(dev)
    # ---- timed region (device events, max over ranks) ----------------------
    # live CUDA-event durations of the dominant kernel only (k_entropy): the
    # roofline needs them from the timed region; bracketing every launch
    # would add host work to every step (--profile-all for the full set)
    if not args.profile_all:
        loader.set_option(N.ESSL_OPT_PROFILE_KERNELS, 1 << N.ESSL_K_ENTROPY)
    loader.set_option(N.ESSL_OPT_PROFILE, 1)
    loader.profile_read()
    launches0 = loader.launches
    pend = []
    if sched:
        loader.retarget(res=sched[0])
    if ws > 1:
        dist.barrier()
    import gc
    gc.collect()
    gc.freeze()  # long-lived objects (torch, numpy) out of the cyclic GC's way
    torch.cuda.synchronize(dev)
    clk.mark()
    prof_range = os.environ.get("ESSL_PROFILER_RANGE") == "1"  # ncu --replay-mode app-range
    if prof_range:
        torch.cuda.cudart().cudaProfilerStart()
    host_t = []
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("bench.timed")
    t0.record(stream)
    n_img = 0
    def stage_of(i):  # progressive stages: equal shares of the timed steps
        return min(len(sched) - 1, i * len(sched) // args.steps) if sched else 0

    i = sets = 0
    while i < args.steps:
        h0 = time.perf_counter()
        if sched:
            r_i = sched[stage_of(i)]
            if r_i != loader.config.res:
                loader.retarget(res=r_i)
        # (as Loader.epochs: single batches until `streams` sets are in flight)
        ps, k = issue(args.warmup + i, args.warmup + args.steps, lambda j: stage_of(j - args.warmup),
                      G if sets >= args.streams else 1)
        sets += 1
        pend.extend(ps)
        n_img += sum(len(p.indices) for p in ps)
        i += k
        h1 = time.perf_counter()
        while len(pend) > 2 * args.streams * G:  # bounded run-ahead; statuses checked as we go
            loader.finish(pend.pop(0))
        host_t.append((h1 - h0, time.perf_counter() - h1))
    for p in pend:  # join every in-flight batch before the end event
        loader.join(p)
    t1.record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize(dev)
    if prof_range:
        torch.cuda.cudart().cudaProfilerStop()
    clk.mark()
    if ws > 1:
        dist.barrier()
    clk.__exit__(None, None, None)
    for p in pend:
        loader.finish(p)
    if True:  # diagnostics on stderr
        ht = np.array(host_t) * 1e3
        log(f"[bench] host enqueue ms median {np.median(ht[:, 0]):.3f} max {ht[:, 0].max():.3f}; "
            f"finish-wait median {np.median(ht[:, 1]):.3f} max {ht[:, 1].max():.3f} "
            f"(argmax {int(ht[:, 0].argmax())}, {int(ht[:, 1].argmax())})")
    ms = t0.elapsed_time(t1)
    launches = loader.launches - launches0
    prof = loader.profile_read()
    loader.set_option(N.ESSL_OPT_PROFILE, 0)
    clocks = clk.summary()
    # ---- e2e: public API, host-staged payloads ------------------------------
    e2e_v = None
    h2d = d2h = 0
    if not args.no_e2e:
        cfg2 = E.LoaderConfig(**{**cfg.__dict__, "resident": False, "staging": args.staging,
                                 **({"fill_chain": args.fill_chain} if args.fill_chain >= 0 else {})})
        l2 = E.Loader(cfg2, container=handle, engine=loader.engine)
        apply_options(l2)
        if args.gather_ctas >= 0:
            l2.set_option(N.ESSL_OPT_GATHER_CTAS, args.gather_ctas)
        if args.gather_tma >= 0:
            l2.set_option(N.ESSL_OPT_GATHER_TMA, args.gather_tma)
        # warm every stream's staging slots and output ring (across epoch
        # boundaries: small shards have fewer batches per epoch than streams)
        for k, b in enumerate(l2.epochs(100)):
            if k + 1 >= 3 * cfg.streams + 3:
                break
        torch.cuda.synchronize(dev)
        if ws > 1:
            dist.barrier()
        n2 = 0
        perm2 = []
        e2e_host = []
        ep = 2
        # as many batches as the device-side timed region, through the public
        # multi-epoch iterator (prefetch kept full across epoch boundaries)
        n_ep = -(-args.steps * B // max(1, len(handle) // ws))
        for e in range(ep, ep + n_ep + 1):  # (bookkeeping for the byte count only)
            perm2.append(E.shard(E.epoch_permutation(cfg.seed, e, len(handle)), rank, ws))
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        hprev = time.perf_counter()
        # exactly `steps` batches are issued (no run-ahead past the timed work)
        for b in l2.epochs(ep, steps=args.steps):
            n2 += len(b)
            now = time.perf_counter()
            e2e_host.append(now - hprev)
            hprev = now
        perm2 = np.concatenate(perm2)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = s0.elapsed_time(s1)
        steps_e2e = max(1, n2 // B)
        lens = handle.records["payload_length"][perm2[:n2]].astype(np.int64)
        h2d = int(lens.sum()) // steps_e2e + B * (ctypes_sizeof_sample() + 24) + 8 * B * 2
        if True:  # diagnostics on stderr (the JSON line is stdout)
            eh = np.array(e2e_host) * 1e3
            log(f"[bench] e2e per-batch host ms median {np.median(eh):.3f} max {eh.max():.3f} "
                f"(argmax {int(eh.argmax())})")
        d2h = B * 32
        e2e_v = (n2, e2e_ms)
    # ---- reduce over ranks ---------------------------------------------------
    from paper_2404_00509_b200.ddp import reduce_timing
    ms_max, total, e2e_ms_max, e2e_total = reduce_timing(
        [ms, n_img, e2e_v[1] if e2e_v else 0.0, e2e_v[0] if e2e_v else 0.0], device=dev)
    if rank == 0:
        value = total / (ms_max / 1e3)
        pk = peaks()
        def bytes_out(r):
            b = 3 * r * r * 2
            if wl["mask"] > 0:
                T = (r // 16) ** 2
                k = int(np.floor(wl["mask"] * T + 0.5))
                b += k * 4 + (T - k) * 8 + T * 8
            return b
        stages = wl.get("schedule") or (res,)
        per_img = float(np.mean(handle.records["payload_length"])) + \
            float(np.mean([bytes_out(r) for r in stages]))
        roof = roofline_block(args, prof, ms, n_img, per_img, value, clocks, pk)
        cpu = None
        if not args.no_cpu:
            cpu = cpu_oracle_rate(path, wl, args.cpu_seconds)
        line = {"metric": METRIC, "value": value, "unit": "images/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "int32", "out_dtype": "bf16", "data": "synthetic",
                "config": config_dict(args, wl, len(handle),
                                      float(np.mean(handle.records["payload_length"]))),
                "roofline": roof, "cpu_baseline": cpu,
                "e2e": {"value": e2e_total / (e2e_ms_max / 1e3) if e2e_v else None,
                        "unit": "images/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
                "gpu_launches": launches, "clocks": clocks}
        print(json.dumps(line), flush=True)
    loader.close()
    if ws > 1:
        dist.destroy_process_group()


def _profile(name: str) -> dict | None:
    """A committed ncu summary (profiles/), newest round first."""
    for tag in ("r2", "r1"):
        p = ROOT / "profiles" / f"{tag}_{name}.json"
        if p.exists():
            d = json.loads(p.read_text())
            d["_src"] = str(p.relative_to(ROOT))
            return d
    return None


def roofline_block(args, prof: dict, ms: float, n_img: int, per_img: float, value: float,
                   clocks: dict, pk: dict) -> dict:
    """HBM roofline of the path: algorithmic bytes per image =
    payload in + bf16 NCHW out (+ mask/ids).  frac: the dominant kernel
    (k_entropy) per the contract -- algorithmic bytes of one launch / its mean
    CUDA-event launch duration inside the timed region (a latency figure:
    8 batches overlap); job_frac: whole-job bytes / time; issue_frac: the
    binding resource, warp instructions per image (pipeline-range ncu) x
    img/s over the issue slots (148 SMs x 4 schedulers x clock); per kernel:
    the isolated ncu launch (256 images) against the same bytes."""
    peak = pk["hbm_gbs"]
    ent_ms, ent_n = prof.get("entropy", (0.0, 0))
    ipl = n_img / max(ent_n, 1)
    achieved = per_img * ipl / (ent_ms / max(ent_n, 1) / 1e3) / 1e9 if ent_n else None
    ent = _profile("ncu_k_entropy") if args.workload == "cfg2" else None
    rng = _profile("ncu_pipeline_range") if args.workload == "cfg2" else None
    sm_hz = (clocks.get("sm_mhz") or 0) * 1e6 or (rng or {}).get("sm_clock_ghz", 1.965) * 1e9
    wipi = (rng or {}).get("warp_instructions_per_image")
    roof = {"bound": "hbm", "kernel": "k_entropy", "achieved": achieved, "peak": peak,
            "peak_src": pk["src"], "unit": "GB/s", "frac": achieved / peak if achieved else None,
            "traffic": (ent or {}).get("dram_bytes"),
            "traffic_src": f"{ent['_src']} (dram read+write bytes of one 256-image launch)" if ent else None,
            "bytes_per_image": per_img, "images_per_launch": ipl,
            "job_achieved": per_img * value / 1e9,
            "job_frac": per_img * value / 1e9 / peak,
            "traffic_pipeline_per_image": (rng or {}).get("dram_bytes_per_image"),
            "issue_frac": wipi * value / (148 * 4 * sm_hz) if wipi else None,
            "warp_instructions_per_image": wipi,
            "issue_src": f"{rng['_src']} x value / (148 SMs x 4 x {sm_hz / 1e6:.0f} MHz)" if rng else None,
            "kernel_ms": {k: v[0] / max(v[1], 1) for k, v in prof.items()},
            "kernel_share": {k: v[0] / ms for k, v in prof.items() if k != "decode"},
            "kernels_isolated": {}}
    if args.workload == "cfg2":
        for k in ("k_prep", "k_entropy", "k_idct", "k_resize", "k_mask"):
            d = _profile(f"ncu_{k}")
            if d and d.get("duration_ns"):
                imgs = 256
                roof["kernels_isolated"][k] = {
                    "us": d["duration_ns"] / 1e3, "images": imgs,
                    "frac": per_img * imgs / (d["duration_ns"] * 1e-9) / 1e9 / peak,
                    "warp_instructions_per_image": d.get("warp_instructions", 0) / imgs,
                    "dram_bytes_per_image": d.get("dram_bytes", 0) / imgs, "src": d["_src"]}
    return roof


def ctypes_sizeof_sample():
    import ctypes

    from paper_2404_00509_b200 import _native as N
    return ctypes.sizeof(N.EsslSample)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--epoch", action="store_true",
                    help="time one full epoch of this rank's shard (steps = batches per epoch)")
    ap.add_argument("--pool", type=int, default=8192)
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--ref-loader-seconds", type=float, default=6.0,
                    help="reference arm: bounded sample per reference-Loader measurement (0: skip)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--seq-bits", type=int, default=0, help="speculative subsequence bits (0: library default)")
    ap.add_argument("--ck-bits", type=int, default=0,
                    help="minimum checkpoint spacing in bits (ESSL_OPT_CHECKPOINT_BITS; 0: default)")
    ap.add_argument("--warm-bits", type=int, default=-1, help="entropy-decode lane warm-up bits (-1: default)")
    ap.add_argument("--stage-bytes", type=int, default=-1,
                    help="ESSL_OPT_STAGE_BYTES (0: entropy lanes read the clean stream from global)")
    ap.add_argument("--resize-cols", type=int, default=0,
                    help="k_resize output columns per thread (ESSL_OPT_RESIZE_COLS; 0: default)")
    ap.add_argument("--resize-band", type=int, default=0,
                    help="k_resize output rows per CTA, at most (ESSL_OPT_RESIZE_BAND; 0: default)")
    ap.add_argument("--profile-all", action="store_true",
                    help="bracket every launch with CUDA events in the timed region (kernel_ms of all kernels)")
    ap.add_argument("--early-exit", type=int, default=-1,
                    help="ESSL_OPT_EARLY_EXIT (entropy decode stops near the crop's last row; -1: default)")
    ap.add_argument("--fill-chain", type=int, default=-1,
                    help="e2e: LoaderConfig.fill_chain (-1: the loader default)")
    ap.add_argument("--group", type=int, default=0,
                    help="consecutive batches decoded per launch set (LoaderConfig.group; "
                         "0: the workload's, 2 unless it sets one)")
    ap.add_argument("--streams", type=int, default=8,
                    help="batches in flight (one libessl context + CUDA stream each)")
    ap.add_argument("--gather-ctas", type=int, default=-1,
                    help="e2e: k_host_gather CTAs (ESSL_OPT_GATHER_CTAS; -1: library default)")
    ap.add_argument("--gather-tma", type=int, default=-1,
                    help="e2e: 1 = bus-read gather with bulk (TMA) copies (ESSL_OPT_GATHER_TMA)")
    ap.add_argument("--staging", default="gather", choices=["gather", "copy"],
                    help="e2e host staging: bus-read gather kernel or host threads + one copy")
    ap.add_argument("--restart", type=int, default=0,
                    help="JPEGs with a restart marker every N MCUs (SURVEY 8(f) f3 variant; "
                         "0: none, as the reference builder)")
    ap.add_argument("--batch", type=int, default=0,
                    help="images per step (0: the workload's batch; analysis knob)")
    ap.add_argument("--aug", default="simple", choices=["simple", "3aug", "3aug+"],
                    help="augmentation level (finetune schemes use 3aug / 3aug+)")
    args = ap.parse_args()
    wl = dict(WORKLOADS[args.workload])
    if args.batch > 0:
        wl["batch"] = args.batch
    if args.group <= 0:
        args.group = wl.get("group", 2)
    if args.restart > 0:
        wl["restart"] = args.restart
        wl["desc"] += f"; restart interval {args.restart} MCUs (f3 variant)"
    if args.aug != "simple":
        wl["aug"] = args.aug
        wl["desc"] = wl["desc"].replace("+ flip +", f"+ flip + {args.aug} +")
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        from paper_2404_00509_b200 import build as B
        B.build()
        run_gpu(args, wl)


if __name__ == "__main__":
    main()
