"""Benchmark: checkpoint save + restore throughput of the B200 data path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c3|c4|c5]
                    [--layers L] [--dir /dev/shm/tvbench] [--impl ours|reference]

Default workload (BASELINE.json configs[1], "C2"): Llama-3-8B-shaped state — bf16
params + fp32 Adam mu/nu, 873 leaves, 80,302,612,480 bytes — FSDP-sharded on dim 0 over
the N GPUs (one logical process per GPU), synthetic random values generated on device.
One step = an asynchronous ``save_checkpoint`` (Orbax's training default: the blocking
device snapshot, then ``wait()`` for pack/D2H/write/commit on /dev/shm; ``--save-mode
sync`` for the zero-copy synchronous save) followed by a
``load_checkpoint`` of the same checkpoint (call → every shard resident in HBM).

value = 2 × tree bytes / step time (GB/s; each byte is saved once and restored once),
time with CUDA events on the current stream bracketing the step, barrier +
synchronize on both sides, max over ranks.  Inputs (80 GB) are far larger than L2.

The JSON line also reports save / restore GB/s separately, the async-save blocking time
against the sync save time, the binding I/O roofline measured in the same run
(min of pinned PCIe D2H/H2D and a pwrite/pread storage probe on the same directory),
the box-copy kernel against the measured HBM copy peak, an end-to-end number through
the host-array API (H2D of the inputs and D2H of the restored arrays inside the timed
region), and the CPU baseline (the oracle port of the reference on a bounded sample).

``--impl reference`` times the reference's CPU path (the oracle port in oracle/, with
one thread per simulated process) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TREE_BYTES_C2 = 80_302_612_480

LLAMA3_8B = dict(layers=32, d=4096, ffn=14336, vocab=128256, kv=1024)


def llama_leaves(layers: int, d: int, ffn: int, vocab: int, kv: int):
    """[(tree, path, shape, dtype)] of the C2 state."""
    shapes = [("embed", (vocab, d)), ("lm_head", (vocab, d)), ("final_norm", (d,))]
    for i in range(layers):
        p = f"layers/{i}"
        shapes += [
            (f"{p}/attn/q", (d, d)), (f"{p}/attn/k", (kv, d)), (f"{p}/attn/v", (kv, d)),
            (f"{p}/attn/o", (d, d)), (f"{p}/mlp/gate", (ffn, d)), (f"{p}/mlp/up", (ffn, d)),
            (f"{p}/mlp/down", (d, ffn)), (f"{p}/norm_in", (d,)), (f"{p}/norm_post", (d,)),
        ]
    out = []
    for tree, dtype in (("params", "bf16"), ("mu", "f32"), ("nu", "f32")):
        out += [(tree, path, shape, dtype) for path, shape in shapes]
    return out


def nbytes(shape, dtype) -> int:
    return math.prod(shape) * (2 if dtype == "bf16" else 4)


# -- environment / measurement helpers ---------------------------------------------------------


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms (rank 0), on the GPUs
    the job uses only: nvidia-smi ignores CUDA_VISIBLE_DEVICES, and idle neighbours on a
    larger box would drag the median toward their idle clock.  GPUs are matched by PCI
    address (some boxes redact nvidia-smi's UUIDs)."""

    QUERY = ("pci.bus_id,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, n_devices: int = 1):
        self.proc = None
        self.path = tempfile.mktemp(prefix="tv_clocks_", suffix=".csv")
        self.buses = set()
        try:
            import torch
            for i in range(min(max(1, n_devices), torch.cuda.device_count())):
                pr = torch.cuda.get_device_properties(i)
                self.buses.add((pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id))
        except Exception:
            self.buses = set()

    @staticmethod
    def _bus(text: str):
        """"00000000:D1:00.0" -> (domain, bus, device)."""
        try:
            dom, bus, dev = text.split(".")[0].split(":")
            return int(dom, 16), int(bus, 16), int(dev, 16)
        except ValueError:
            return None

    def start(self):
        if shutil.which("nvidia-smi") is None:
            return
        self.f = open(self.path, "w")
        self.proc = subprocess.Popen(
            ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits", "-lms", "200"],
            stdout=self.f, stderr=subprocess.DEVNULL)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        rows = [[p.strip() for p in line.split(",")] for line in open(self.path)]
        mine = [r for r in rows if len(r) >= 9 and self._bus(r[0]) in self.buses]
        if not mine:  # PCI addresses unresolved: sample every GPU on the box
            self.buses = set()
            mine = rows
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for parts in mine:
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(name)
        os.unlink(self.path)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
            "gpus_sampled": len(self.buses) or "all",
        }


def measured_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class Dist:
    """torchrun plumbing of the bench: NCCL process group, one rank per GPU.  When there
    are more local ranks than GPUs (a robustness run of the 8-rank path on a smaller box)
    ranks share GPUs round-robin and the bench's own collectives go over gloo (NCCL
    refuses two ranks on one GPU)."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.local = self.local_rank
        self.on = self.world > 1
        self.dev = "cuda"

    def init(self):
        import datetime

        import torch
        import torch.distributed as dist

        n = max(1, torch.cuda.device_count())
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(self.world)))
        self.local = self.local_rank % n
        if self.on and not dist.is_initialized():
            torch.cuda.set_device(self.local)
            if local_world > n:
                self.dev = "cpu"
                dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=1800))
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local),
                                        timeout=datetime.timedelta(seconds=1800))

    def barrier(self):
        if self.on:
            import torch.distributed as dist

            if dist.is_initialized():
                dist.barrier()

    def _reduce(self, x: float, op) -> float:
        import torch
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x: float) -> float:
        if not self.on:
            return x
        import torch.distributed as dist

        return self._reduce(x, dist.ReduceOp.MAX)

    def sum(self, x: float) -> float:
        if not self.on:
            return x
        import torch.distributed as dist

        return self._reduce(x, dist.ReduceOp.SUM)


# -- workload ------------------------------------------------------------------------------------


def gen_shard(i: int, tree: str, dtype: str, ranges, seed: int, gpu: int):
    """The synthetic values of leaf ``i``'s box ``ranges`` (a shard), generated on ``gpu``:
    N(0, 0.02) params, N(0, 1e-3) mu, N(0, 1e-3)^2 nu, seeded by the leaf and the box's
    first row (replicas of a range hold identical values).  Deterministic, so any rank
    can regenerate any shard to verify a restore against."""
    import torch

    with torch.cuda.device(gpu):
        gen = torch.Generator(device=f"cuda:{gpu}")
        gen.manual_seed(1000 * (i + 1) + (ranges[0][0] if ranges else 0) + seed)
        ext = tuple(e for _, e in ranges)
        t = torch.empty(ext, dtype=torch.float32 if dtype == "f32" else torch.bfloat16, device=f"cuda:{gpu}")
        t.normal_(0.0, 0.02 if tree == "params" else 1e-3, generator=gen)
        if tree == "nu":
            t.mul_(t)
    return t


def build_state(tv, rt, mesh, leaves, seed=0, spec_fn=None):
    """Device shards of every leaf for the devices this process owns (``gen_shard``)."""
    import torch

    trees, shardings = {}, {}
    owned = set(rt.addressable_processes)
    for i, (tree, path, shape, dtype) in enumerate(leaves):
        spec = (spec_fn or (lambda s: ("fsdp",) + (None,) * (len(s) - 1)))(shape)
        node = trees.setdefault(tree, {})
        parts = path.split("/")
        for p in parts[:-1]:
            node = node.setdefault(p, {})
        if spec is None:  # unsharded leaf: one global array on process 0's GPU
            gpu = rt.gpu_of_process(0)
            node[parts[-1]] = tv.DenseArray(dtype, gen_shard(i, tree, dtype, tuple((0, e) for e in shape),
                                                             seed, gpu))
            continue
        s = tv.Sharding(mesh, tv.PartitionSpec(spec), shape)
        shards = {}
        for sh in tv.shards_of(s):
            if mesh.process_of(sh.device) not in owned:
                continue
            shards[sh.device] = gen_shard(i, tree, dtype, sh.ranges, seed, rt.gpu_of_device(sh.device))
        node[parts[-1]] = tv.ShardedArray(dtype, s, shards)
        shardings.setdefault(tree, {})[path] = s
    torch.cuda.synchronize()
    return {"state": trees}, {"state": _flatten_shardings(shardings)}


def _flatten_shardings(per_tree):
    out = {}
    for tree, per in per_tree.items():
        for path, s in per.items():
            out[f"{tree}/{path}"] = s
    return out


METRIC = "checkpoint save+restore throughput (GB/s of tree bytes, save and restore each count once)"


def bench_config(args, N: int) -> dict:
    """The ``config`` object of BOTH arms' JSON lines: what workload the line measures
    (tree, mesh, save mode, storage target) and nothing about how an arm runs it, so the
    two lines of one configuration compare equal."""
    if args.config == "c1":
        workload = "C1 4 x (4096,4096) f32 unsharded (268435456 bytes), process 0 writes"
        tree_bytes, layers = 4 * 4096 * 4096 * 4, 0
    else:
        leaves = llama_leaves(**dict(LLAMA3_8B, layers=args.layers))
        tree_bytes, layers = sum(nbytes(s, dt) for _, _, s, dt in leaves), args.layers
        mesh = {"c2": f"FSDP-{N} on dim 0", "c3": f"2x{N // 2} (replica x fsdp) mesh, replica-parallel save",
                "c3ss": f"2x{N // 2} (replica x fsdp) mesh, single-slice save",
                "c4": f"saved 1x{N} (FSDP-{N}) -> restored onto 2x{(args.restore_gpus or N) // 2} "
                      f"(replica x fsdp)"}.get(args.config, args.config)
        workload = (f"{args.config.upper()} Llama-3-8B bf16 params + fp32 Adam mu/nu, {len(leaves)} leaves, "
                    f"{tree_bytes} bytes, {mesh}")
    return {
        "workload": workload + f"; {args.save_mode} save -> restore per step, {args.layout} layout",
        "config": args.config,
        "layers": layers,
        "tree_bytes": tree_bytes,
        "storage": "tmpfs huge=always" if args.storage == "hugetmpfs" else "tmpfs /dev/shm",
        "parallelism": f"{N} GPU(s), one logical process per GPU",
        "l2": "inputs (tree bytes) far larger than the 126 MB L2; no flush needed",
    }


class Workload:
    """One benchmark configuration (BASELINE.json configs)."""

    def __init__(self, tv, name, leaves, save_mesh, spec_fn, save_options, restore_mesh=None,
                 restore_P=None, describe=""):
        self.tv, self.name, self.leaves = tv, name, leaves
        self.save_mesh, self.spec_fn, self.save_options = save_mesh, spec_fn, save_options
        self.restore_mesh = restore_mesh          # None: restore onto the saved topology
        self.restore_P = restore_P
        self.describe = describe
        self.tree_bytes = sum(nbytes(s, dt) for _, _, s, dt in leaves)

    def shardings(self, mesh):
        tv = self.tv
        out = {}
        for tree, path, shape, dtype in self.leaves:
            spec = self.spec_fn(shape)
            out[f"{tree}/{path}"] = None if spec is None else tv.Sharding(mesh, tv.PartitionSpec(spec), shape)
        return out

    def abstract(self):
        tv = self.tv
        sh = self.shardings(self.restore_mesh)
        tree: dict = {}
        for t, path, shape, dtype in self.leaves:
            node = tree.setdefault(t, {})
            parts = path.split("/")
            for p in parts[:-1]:
                node = node.setdefault(p, {})
            node[parts[-1]] = tv.AbstractLeaf("array", shape, dtype, sh[f"{t}/{path}"])
        return {"state": tree}


def fsdp_spec(shape):
    return ("fsdp",) + (None,) * (len(shape) - 1)


def make_workload(tv, args, N) -> Workload:
    dims = dict(LLAMA3_8B, layers=args.layers)
    llama = llama_leaves(**dims)
    cfg = args.config
    if cfg == "c1":
        leaves = [("model", f"a{i}", (4096, 4096), "f32") for i in range(4)]
        mesh = tv.Mesh.create([("solo", 1)], process_count=1)
        return Workload(tv, "c1", leaves, mesh, lambda s: None, tv.SaveOptions(sync=True, layout=args.layout),
                        describe="C1 4 x (4096,4096) f32 unsharded, process 0 writes, " + args.save_mode + " save -> restore")
    if cfg == "c2":
        mesh = tv.Mesh.create([("fsdp", N)], process_count=N)
        return Workload(tv, "c2", llama, mesh, fsdp_spec, tv.SaveOptions(sync=True, layout=args.layout),
                        describe=f"C2 Llama-3-8B bf16 params + fp32 Adam mu/nu, FSDP-{N} on dim 0, "
                                 f"{args.save_mode} save -> restore, {args.layout} layout")
    if cfg in ("c3", "c3ss"):
        if N % 2:
            raise SystemExit("c3 needs an even number of GPUs (replica 2 x fsdp N/2)")
        mesh = tv.Mesh.create([("replica", 2), ("fsdp", N // 2)], process_count=N, replica_axis="replica")
        rp = cfg == "c3"
        return Workload(tv, cfg, llama, mesh, fsdp_spec,
                        tv.SaveOptions(sync=True, replica_parallel=rp, layout=args.layout),
                        describe=f"C3 Llama-3-8B on a 2x{N // 2} (replica x fsdp) mesh, "
                                 f"{'replica-parallel' if rp else 'single-slice'} {args.save_mode} save -> restore")
    if cfg == "c4":
        if N % 2:
            raise SystemExit("c4 needs an even number of GPUs")
        Pr = args.restore_gpus or N
        save_mesh = tv.Mesh.create([("fsdp", N)], process_count=N)
        rmesh = tv.Mesh.create([("replica", 2), ("fsdp", Pr // 2)], process_count=Pr, replica_axis="replica")
        return Workload(tv, "c4", llama, save_mesh, fsdp_spec, tv.SaveOptions(sync=True, layout=args.layout),
                        restore_mesh=rmesh,
                        restore_P=Pr,
                        describe=f"C4 Llama-3-8B saved 1x{N} (FSDP-{N}) -> restored onto 2x{Pr // 2} "
                                 f"(replica x fsdp, {Pr} GPUs), read-once + NVLink fan-out")
    raise SystemExit(f"unknown config {cfg}")


def prepare_storage(args, d) -> str:
    """Storage target: ``hugetmpfs`` (default) = a tmpfs mounted with huge=always for this
    run on the same host RAM as /dev/shm (2 MiB pages cut the per-page cost of page-cache
    writes: measured +25-40 % pwrite, +35 % pread on these boxes, profiles/
    r01_storage_shm_vs_hugetmpfs.txt), falling back to /dev/shm when it cannot be mounted
    (not root, no mount binary); ``shm`` = /dev/shm.  The roofline probe always runs on
    the target actually used, and ``config.storage`` names it."""
    if args.storage == "shm":
        return args.dir
    mnt = "/mnt/tvbench_huge"
    if d.rank == 0:
        try:
            os.makedirs(mnt, exist_ok=True)
            if not os.path.ismount(mnt):
                total_kb = int(open("/proc/meminfo").read().split("MemTotal:")[1].split()[0])
                size = int(total_kb * 0.8)
                rc = subprocess.run(["mount", "-t", "tmpfs", "-o", f"size={size}k,huge=always", "tmpfs", mnt],
                                    capture_output=True).returncode
                if rc == 0:
                    import atexit

                    atexit.register(lambda: subprocess.run(["umount", "-l", mnt], capture_output=True))
        except OSError:
            pass
    d.barrier()
    if not os.path.ismount(mnt):
        print(f"bench: cannot mount a huge-page tmpfs at {mnt}; using {args.dir}", file=sys.stderr)
        args.storage = "shm"
        return args.dir
    return os.path.join(mnt, "tvbench")


def open_runtime(tv, d, N, backend, gpus=None):
    import torch

    if d.on:
        return tv.DistributedRuntime(backend)
    visible = torch.cuda.device_count()
    gpus = [g for g in (gpus if gpus is not None else range(N)) if g < visible] or [0]
    return tv.SimulatedRuntime(N, backend, gpus=gpus)


def _numa_nodes() -> int:
    import glob

    from paper_2605_23066_b200 import native

    n = 0
    for node in glob.glob("/sys/devices/system/node/node[0-9]*"):
        try:
            with open(f"{node}/cpulist") as f:
                n += bool(native.parse_cpulist(f.read()))
        except OSError:
            pass
    return n


def run_ours(args) -> dict:
    import torch

    import paper_2605_23066_b200 as tv
    from paper_2605_23066_b200 import native
    from paper_2605_23066_b200.training_manager import delete_checkpoint

    d = Dist()
    d.init()
    N = d.world if d.on else args.gpus
    torch.cuda.set_device(d.local)
    base = prepare_storage(args, d)
    if d.rank == 0:
        shutil.rmtree(base, ignore_errors=True)
        os.makedirs(base, exist_ok=True)
    d.barrier()
    # the main loop is throughput-bound steady-state checkpointing of one tree: recycled
    # files are registered with CUDA (once each, during warm-up) for zero-copy DMA
    backend = tv.FilesystemBackend(base, register_pool=bool(args.recycle) and not args.no_register)
    wl = make_workload(tv, args, N)
    P = wl.save_mesh.process_count
    rt = open_runtime(tv, d, P, backend, gpus=list(range(N)))
    rrt = rt
    if wl.restore_P is not None and wl.restore_P != P:
        if d.on:
            # restore onto fewer ranks than saved (C4 "saved on 8, restored onto 4"): the
            # first restore_P ranks form the restoring job; the others sit the restore out
            if wl.restore_P > d.world:
                raise SystemExit(f"--restore-gpus {wl.restore_P} > {d.world} ranks")
            rrt = tv.DistributedRuntime.subgroup(backend, list(range(wl.restore_P)))
        else:
            rrt = tv.SimulatedRuntime(wl.restore_P, backend, gpus=list(range(min(N, wl.restore_P))))
    state, shardings = build_state(tv, rt, wl.save_mesh, wl.leaves, spec_fn=wl.spec_fn)
    abstract = wl.abstract() if wl.restore_mesh is not None else None
    torch.cuda.synchronize()
    tree_bytes = wl.tree_bytes

    import dataclasses

    sync_opts = dataclasses.replace(wl.save_options, sync=True)
    async_opts = dataclasses.replace(wl.save_options, sync=False)
    step_opts = async_opts if args.save_mode == "async" else sync_opts

    timing = False
    ksave = {"ms_total": 0.0, "ms_max": 0.0, "bytes": 0, "launches": 0}
    kload = dict(ksave)

    def _add(acc, k):
        acc["ms_total"] += k["ms_total"]
        acc["ms_max"] = max(acc["ms_max"], k["ms_max"])
        acc["bytes"] += k["bytes"]
        acc["launches"] += k["launches"]

    verified = {}
    step_snap: list[float] = []

    def step(i: int, opts=None, verify: bool = False):
        """One save (call -> committed) + one restore (call -> every shard resident).
        Async mode (Orbax's default for training): the blocking device snapshot, then
        wait() for the background pack/D2H/write/commit.  Returns (save ms, restore ms,
        save wall ms, restore wall ms, blocking ms)."""
        opts = opts or step_opts
        path = f"bench/step_{i:04d}"
        d.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev2 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ev0.record()
        handle = tv.save_checkpoint(rt, path, state, shardings, opts)
        tb = time.perf_counter()
        handle.wait()
        ev1.record()
        t1 = time.perf_counter()
        if timing:
            ks = native.kernel_timing_collect()
            _add(ksave, ks)
            step_snap.append(ks["ms_max"])  # this step's device snapshot (async mode)
        if abstract is None:
            out = tv.load_checkpoint(rt, path, None, tv.LoadOptions(), current_mesh=wl.save_mesh)
        elif rrt is not None:
            out = tv.load_checkpoint(rrt, path, abstract, tv.LoadOptions())
        else:  # this rank is outside the restoring job
            out = None
        ev2.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if timing:
            _add(kload, native.kernel_timing_collect())
        if verify:  # outside every timed number: restored bytes == saved state, on device
            nb, bad = verify_restore(tv, state, out, wl.leaves) if out is not None else (0, 0)
            verified["bytes_compared"] = int(d.sum(nb))
            verified["mismatched_boxes"] = int(d.sum(bad))
        del out
        # retire the checkpoint (counted in the step): process 0 deletes it as retention
        # would — with recycling, its chunk files go to the recycle pool and the next
        # save overwrites them in place (steady-state checkpointing with max_to_keep)
        d.barrier()
        tr = time.perf_counter()
        retire_checkpoint(d, backend, path, args.recycle)
        if d.rank == 0:
            shutil.rmtree(os.path.join(base, path), ignore_errors=True)  # emptied dirs
        retire_ms = d.max((time.perf_counter() - tr) * 1e3)
        d.barrier()
        return (ev0.elapsed_time(ev1), ev1.elapsed_time(ev2), (t1 - t0) * 1e3, (t2 - t1) * 1e3,
                (tb - t0) * 1e3, retire_ms)

    for i in range(args.warmup):
        step(i)

    # roofline probes in the same run and directory, after warm-up (a VM's first touch of
    # fresh memory is slower than steady state)
    probe = {}
    if d.rank == 0:
        nthreads = min(128, len(os.sched_getaffinity(0)))
        best = (0.0, 0.0, 0.0)
        for _ in range(2):
            w_gbs, rw_gbs, r_gbs = native.probe_storage_rewrite(base, nthreads, 1 << 30, 8 << 20)
            best = (max(best[0], w_gbs), max(best[1], rw_gbs), max(best[2], r_gbs))
        probe["storage_write_fresh_GBps"] = round(best[0], 2)
        probe["storage_rewrite_GBps"] = round(best[1], 2)
        # the save's storage roofline: fresh files, or files rewritten in place when the
        # save overwrites recycled files
        probe["storage_write_GBps"] = round(best[1] if args.recycle else best[0], 2)
        probe["storage_read_GBps"] = round(best[2], 2)
        probe["storage_threads"] = nthreads
        probe["storage_probe"] = (f"{nthreads} threads x 1 GiB files, 8 MiB pwrite/pread from pinned memory, "
                                  "best of 2; write = " + ("rewrite of existing files (recycling on)"
                                                           if args.recycle else "fresh files"))
    d.barrier()  # every rank probes its own link at the same time: the aggregate is concurrent
    # 3 rounds of (one warm-up + one timed 4 GiB copy per direction), every rank at once
    # after a barrier, mean of the rounds: the ranks' copies overlap, so the sum over ranks
    # is what the GPUs get concurrently (best of 3 x 1 GiB let a rank time a copy that ran
    # partly alone, overstating the aggregate)
    rounds = []
    for _ in range(3):
        d.barrier()
        rounds.append(native.probe_pcie(d.local if d.on else 0, 4 << 30, 1))
    d2h = statistics.mean(r[0] for r in rounds)
    h2d = statistics.mean(r[1] for r in rounds)
    probe["pcie_d2h_GBps_per_gpu"] = round(d2h, 2)
    probe["pcie_h2d_GBps_per_gpu"] = round(h2d, 2)
    if d.on:
        probe["pcie_d2h_GBps_aggregate"] = round(d.sum(d2h), 2)
        probe["pcie_h2d_GBps_aggregate"] = round(d.sum(h2d), 2)
        probe["pcie_aggregate_how"] = ("all ranks' pinned 4 GiB D2H / H2D copies at once after a barrier, "
                                       "mean of 3 rounds per rank, summed over ranks")
    else:
        probe["pcie_d2h_GBps_aggregate"] = round(d2h * N, 2)
        probe["pcie_h2d_GBps_aggregate"] = round(h2d * N, 2)
        probe["pcie_aggregate_how"] = "GPU 0's link x GPUs" if N > 1 else "one GPU"
    # the same storage probe with every rank's copy engine busy at once (D2H during the
    # writes, H2D during the reads): a copy-through-pinned pipeline's DMA and page-cache
    # copies share host memory, so these contended rates are the context of save/restore
    cores = min(128, len(os.sched_getaffinity(0)))
    local_world = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1"))) if d.on else 1
    per_rank = max(1, cores // local_world)
    cdir = os.path.join(base, f"contended_{d.rank}")
    d.barrier()
    cw, cr, cd2h, ch2d = native.probe_storage_dma(cdir, per_rank, 1 << 30, 8 << 20, d.local if d.on else 0)
    shutil.rmtree(cdir, ignore_errors=True)
    contended = {"write_GBps": round(d.sum(cw), 2), "read_GBps": round(d.sum(cr), 2),
                 "d2h_GBps": round(d.sum(cd2h), 2), "h2d_GBps": round(d.sum(ch2d), 2),
                 "how": f"every rank: {per_rank} threads x 1 GiB pwrite/pread on its own files while a DMA "
                        "thread loops 64 MiB D2H (during writes) / H2D (during reads) on its GPU; summed"}
    d.barrier()

    clocks = ClockSampler(max(N, args.restore_gpus or 0))
    if d.rank == 0:
        clocks.start()
    import gc

    gc_ms = [0.0, 0, 0]  # time, collections, gen-2 collections in the timed steps (this rank)
    gc_t0 = [0.0]

    gc_sources: dict[str, list] = {}  # TVGPU_GC_SOURCES=1: where collections are triggered
    trace_gc = os.environ.get("TVGPU_GC_SOURCES") == "1"

    def _gc_cb(phase, info):
        if phase == "start":
            gc_t0[0] = time.perf_counter()
            if trace_gc:
                import traceback

                ours = [f for f in traceback.extract_stack()[:-1]
                        if "paper_2605_23066_b200" in f.filename or f.filename.endswith("bench.py")]
                if ours:
                    f = ours[-1]
                    site = f"{os.path.basename(f.filename)}:{f.lineno} {f.name}"
                    gc_sources.setdefault(site, [0, 0.0])[0] += 1
                    gc_t0.append(site)
        else:
            dt_ms = (time.perf_counter() - gc_t0[0]) * 1e3
            gc_ms[0] += dt_ms
            if len(gc_t0) > 1:
                gc_sources[gc_t0.pop()][1] += dt_ms
            gc_ms[1] += 1
            gc_ms[2] += int(info.get("generation") == 2)

    gc.callbacks.append(_gc_cb)
    before = native.totals()
    native.kernel_timing(True)
    timing = True
    saves, restores, walls, blocks, host_blocks, snaps, retires = [], [], [], [], [], [], []
    for i in range(args.steps):
        s_ms, r_ms, ws, wr, b_ms, rt_ms = step(args.warmup + i)
        saves.append(d.max(s_ms))
        restores.append(d.max(r_ms))
        retires.append(rt_ms)
        walls.append(d.max(ws + wr) + rt_ms)
        host_blocks.append(d.max(b_ms))
        snaps.append(d.max(step_snap[-1]) if args.save_mode == "async" and step_snap else 0.0)
        blocks.append(host_blocks[-1] + snaps[-1])
    native.kernel_timing(False)
    timing = False
    native.kernel_timing_collect()
    gc.callbacks.remove(_gc_cb)
    from paper_2605_23066_b200 import timeline

    me = d.rank if d.on else 0
    phases = {"save": dict(timeline.LAST_SAVE.get(me, {})),
              "restore": {**timeline.LAST_RESTORE.get(me, {}), **timeline.LAST_RESTORE.get(-1, {})}}
    # rank skew: each process's own write phase / engine load in the last step
    mine = {p: [round(ph.get("write_phase", 0.0), 1),
                round(timeline.LAST_RESTORE.get(p, {}).get("engine_load", 0.0), 1)]
            for p, ph in timeline.LAST_SAVE.items()}
    if d.on:
        import torch.distributed as dist

        every = [None] * d.world
        dist.all_gather_object(every, {me: mine.get(me, [0.0, 0.0])})
        mine = {k: v for part in every for k, v in part.items()}
    skew = {"write_phase_ms": [mine[p][0] for p in sorted(mine)],
            "engine_load_ms": [mine[p][1] for p in sorted(mine)]}
    after = native.totals()
    clock_info = clocks.stop() if d.rank == 0 else {}
    kernels = d.sum(after["kernel_launches"] - before["kernel_launches"])
    dmas = d.sum(after["dma_copies"] - before["dma_copies"])
    engine = {}
    for kind in ("save", "load"):
        a, b = after[kind], before[kind]
        wall = max(1e-9, a["seconds_total"] - b["seconds_total"])
        engine[kind] = {
            "wall_s": round(wall, 3),
            "thread_io_s": round(a["seconds_io"] - b["seconds_io"], 3),
            "thread_wait_dma_s": round(a["seconds_wait_dma"] - b["seconds_wait_dma"], 3),
            "producer_wait_slot_s": round(a["seconds_wait_slot"] - b["seconds_wait_slot"], 3),
            "storage_GB": round((a["bytes_storage"] - b["bytes_storage"]) / 1e9, 3),
            "pcie_GB": round((a["bytes_device"] - b["bytes_device"]) / 1e9, 3),
            # save: bytes packed by the kernel; load: bytes the unpack / NVLink fan-out moved
            "kernel_GB": round((a["bytes_packed"] - b["bytes_packed"]) / 1e9, 3),
            # bytes DMA'd straight into / out of registered recycled files (no pinned slot)
            "zero_copy_GB": round((a["zero_copy_bytes"] - b["zero_copy_bytes"]) / 1e9, 3),
        }
    peer_gb = d.sum(after["peer_bytes"] - before["peer_bytes"]) / 1e9
    zc_frac = {}
    for kind in ("save", "load"):
        moved = d.sum(after[kind]["bytes_storage"] - before[kind]["bytes_storage"])
        zc_frac[kind] = d.sum(after[kind]["zero_copy_bytes"] - before[kind]["zero_copy_bytes"]) / max(1, moved)
    save_ms = statistics.mean(saves)
    restore_ms = statistics.mean(restores)
    retire_ms = statistics.mean(retires)
    step_ms = save_ms + restore_ms + retire_ms
    value = 2 * tree_bytes / (step_ms / 1e3) / 1e9
    save_gbs = tree_bytes / (save_ms / 1e3) / 1e9
    restore_gbs = tree_bytes / (restore_ms / 1e3) / 1e9

    snap_dev_ms = statistics.mean(snaps) if args.save_mode == "async" else 0.0
    # async-save blocking vs the synchronous save it replaces: the timed steps give one
    # side, one extra save (untimed for `value`) in the other mode gives the other
    if args.save_mode == "async":
        blocking_ms = statistics.mean(host_blocks)
        other = step(args.warmup + args.steps, sync_opts, verify=True)
        sync_save_ms = d.max(other[0])
        async_total_ms = save_ms
    else:
        sync_save_ms = save_ms
        other = step(args.warmup + args.steps, async_opts, verify=True)
        blocking_ms = d.max(other[4])
        async_total_ms = d.max(other[0])
    d.barrier()
    if d.rank == 0:
        shutil.rmtree(os.path.join(base, "bench"), ignore_errors=True)

    kern = kernel_roofline(tv, native, state, rt, d, ksave, kload, args, step_ms, peer_gb)
    reshard = (reshard_leg(tv, native, d, rt, wl, state, shardings, args, N, base)
               if args.reshard_steps > 0 and wl.name == "c2" else None)
    free_recycle_pool(native, d, backend)  # the main tree's retired files: not needed again
    # the e2e leg is the same steady state through host buffers (its own warm-up registers
    # its files); the C5 loop below recycles without registering: in a training loop the
    # one-time registration would lengthen the first background saves past the step,
    # which is exactly the blocking C5 measures (FilesystemBackend(register_pool=False))
    e2e = end_to_end(tv, rt, wl, args, d, base) if not args.no_e2e else None
    backend.register_pool = False
    free_recycle_pool(native, d, backend)
    c5 = None
    if args.c5_layers > 0 and wl.name == "c2":
        # BASELINE configs[4] in the default line: the training loop's blocking time with a
        # Checkpointer saving every step (its own smaller tree: keep_last=3 + 1 in flight
        # must fit the RAM-backed storage next to nothing else)
        del state
        torch.cuda.empty_cache()
        c5 = c5_loop(tv, d, rt, N, base, args.c5_layers, args.c5_steps, args.train_ms, recycle=args.recycle)
        free_recycle_pool(native, d, backend)
    c3 = (c3_leg(tv, native, d, rt, backend, args, N, base)
          if args.c3_steps > 0 and wl.name == "c2" and N >= 4 and N % 2 == 0 else None)
    c1 = c1_leg(tv, native, d, base, args) if args.c1_steps > 0 and wl.name == "c2" else None

    peaks = measured_peaks()
    result = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": N,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_ms, 2),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u8",
        "payload_dtypes": "bf16 params + f32 Adam mu/nu, moved as bytes (no arithmetic on the path)",
        "data": "synthetic (random values generated on device, Llama-3-8B shapes)",
        "config": bench_config(args, N),
        "arm": {
            "storage_path": base,
            "runtime": "torchrun (DistributedRuntime)" if d.on else "threads (SimulatedRuntime)",
            "timing": "CUDA events on the current stream around save and restore, barrier+sync both sides, "
                      "max over ranks",
        },
        "save_GBps": round(save_gbs, 3),
        "restore_GBps": round(restore_gbs, 3),
        "save_ms": round(save_ms, 2),
        "restore_ms": round(restore_ms, 2),
        "retire_ms": round(retire_ms, 2),
        "recycle": {"enabled": bool(args.recycle),
                    "register_pool": "main C2 loop, e2e and C1 legs (FilesystemBackend(register_pool=True)); the C5 loop recycles without registering",
                    "save_path_rates_rank0": native.SAVE_PATHS.snapshot(),
                    "files_overwritten_in_timed_steps": int(d.sum(after["save"]["recycled_files"]
                                                                  - before["save"]["recycled_files"])),
                    "note": "each step ends by retiring its checkpoint (process 0, inside the timed step); "
                            "with recycling its chunk files go to the backend's recycle pool and the next "
                            "save overwrites them in place (FilesystemBackend .tvpool; steady-state "
                            "checkpointing with max_to_keep) instead of allocating fresh page-cache pages; "
                            "each GPU's saves use whichever of zero-copy (D2H into the registered pages) and "
                            "slot ring + pwrite measured faster on this box (native.SavePathChooser)"},
        "wall_ms_per_step": round(statistics.mean(walls), 2),
        "save_mode": args.save_mode,
        "async_blocking_ms": round(blocking_ms + snap_dev_ms, 2),
        "async_blocking_breakdown": {
            "host_ms": round(blocking_ms, 2),
            "device_snapshot_ms": round(snap_dev_ms, 2),
            "note": "save() returns once the snapshot is enqueued on the caller's stream (host_ms); "
                    "the snapshot kernel then holds that stream for device_snapshot_ms (mean over the "
                    "timed steps) — both are counted as blocking",
        },
        "async_total_ms": round(async_total_ms, 2),
        "sync_save_ms": round(sync_save_ms, 2),
        "async_blocking_frac_of_sync_save": round((blocking_ms + snap_dev_ms) / sync_save_ms, 4),
        "async_blocking_ms_per_step": ({"p50": round(_pct(blocks, 50), 2), "p99": round(_pct(blocks, 99), 2),
                                        "max": round(max(blocks), 2),
                                        "p99_frac_of_sync_save": round(_pct(blocks, 99) / sync_save_ms, 4),
                                        "how": "per timed step: host time in save_checkpoint + that step's "
                                               "snapshot kernel (max over ranks)"}
                                       if args.save_mode == "async" else None),
        "io_roofline": None,
        "roofline": kern,
        "e2e": e2e,
        "c5": c5,
        "c1": c1,
        "c3": c3,
        "reshard": reshard,
        "gpu_launches": int(kernels),
        "gpu_launches_breakdown": {
            "box_copy_kernel": int(kernels),
            "copy_engine_dma_by_libtvgpu": int(dmas),
            "note": "gpu_launches counts libtvgpu kernel launches only (summed over ranks); "
                    "contiguous chunk payloads move by copy-engine DMA issued by libtvgpu's engine "
                    "(measured faster than SM-driven PCIe: profiles/r01_pcie_kernel_vs_ce.jsonl); "
                    "async-save snapshots, strided boxes and reshard scatters run box_copy_kernel",
        },
        "clocks": clock_info,
        "engine_rank0": engine,
        "numa_rank0": {"nodes_with_cpus": _numa_nodes(), **native.placement(),
                       "note": "storage threads + pinned ring bound to the GPU's local CPUs "
                               "when the host has > 1 NUMA node (torchrun); {} = not placed"},
        "phases_ms_rank0_last_step": phases,
        "per_process_last_step": skew,
        "python_gc_rank0": {"ms_per_step": round(gc_ms[0] / args.steps, 2),
                            "collections": gc_ms[1], "gen2": gc_ms[2],
                            **({"sources": sorted(([k, n, round(t, 2)] for k, (n, t) in gc_sources.items()),
                                                  key=lambda x: -x[2])[:25]} if trace_gc else {})},
        "restore_verified": dict(verified, how="after the timed steps: every restored shard's overlap "
                                               "with every saved shard compared with torch.equal on "
                                               "the device (all ranks)"),
        "reshard_exchange": {
            "nvlink_GB_per_restore": round(peer_gb / args.steps, 3),
            "nvlink_GBps_over_restore": round(peer_gb / args.steps / (restore_ms / 1e3), 2),
            "note": "bytes the read-once fan-out kernel stored into OTHER GPUs' HBM (P2P / CUDA IPC "
                    "over NVLink), summed over GPUs, per restore; overlapped with the storage reads",
        },
    }
    if d.rank == 0:
        pcie_d2h = probe["pcie_d2h_GBps_aggregate"]
        pcie_h2d = probe["pcie_h2d_GBps_aggregate"]
        # Bytes a save / restore moved zero-copy (DMA straight into / out of registered
        # page-cache pages) are bound by PCIe alone; the rest by min(storage, PCIe): the
        # step's roofline is the byte-weighted harmonic mix of the two paths.
        zc_save, zc_load = zc_frac["save"], zc_frac["load"]
        save_peak = 1.0 / (zc_save / pcie_d2h + (1 - zc_save) / min(probe["storage_write_GBps"], pcie_d2h))
        restore_peak = 1.0 / (zc_load / pcie_h2d + (1 - zc_load) / min(probe["storage_read_GBps"], pcie_h2d))
        result["io_roofline"] = {
            "bound": ("pcie" if min(zc_save, zc_load) > 0.5 or probe["storage_write_GBps"] >= pcie_d2h
                      else "storage"),
            "zero_copy_fraction": {"save": round(zc_save, 4), "restore": round(zc_load, 4),
                                   "note": "share of bytes DMA'd straight into / out of registered "
                                           "page-cache pages (no pinned slot, no pwrite/pread): bound by "
                                           "PCIe only; the storage probe is the pwrite/pread path's bound"},
            "save_peak_GBps": round(save_peak, 2),
            "restore_peak_GBps": round(restore_peak, 2),
            "save_frac": round(save_gbs / save_peak, 4),
            "restore_frac": round(restore_gbs / restore_peak, 4),
            "step_frac": round(value / (2 / (1 / save_peak + 1 / restore_peak)), 4),
            **probe,
            "contended": dict(contended,
                              save_vs_min_write_d2h=round(save_gbs / max(1e-9, min(contended["write_GBps"],
                                                                                   contended["d2h_GBps"])), 4),
                              restore_vs_min_read_h2d=round(restore_gbs / max(1e-9, min(contended["read_GBps"],
                                                                                        contended["h2d_GBps"])), 4),
                              note="context, not the roofline: both flows at full blast at once (the "
                                   "pipeline moves each byte through both at the same rate)"),
        }
        result["roofline"]["peak_source"] = peaks["source"]
        if not args.no_cpu_baseline and N == 1:  # rank 0 at N=1 only (the contract)
            result["cpu_baseline"] = cpu_baseline(args, root_dir=base)
    return result


def _storage_room(path: str):
    """Bytes the storage under `path` can take: free space, capped by available host RAM
    when the filesystem is RAM-backed (tmpfs)."""
    try:
        st = os.statvfs(path)
        free = st.f_bavail * st.f_frsize
        fstype = ""
        best = ""
        for line in open("/proc/mounts"):
            dev, mnt, typ = line.split()[:3]
            if os.path.realpath(path).startswith(mnt.rstrip("/") + "/") and len(mnt) > len(best):
                best, fstype = mnt, typ
        if fstype in ("tmpfs", "ramfs"):
            for line in open("/proc/meminfo"):
                if line.startswith("MemAvailable:"):
                    free = min(free, int(line.split()[1]) * 1024)
        return free
    except (OSError, ValueError):
        return None


def _pct(xs, q):
    """Nearest-rank percentile."""
    xs = sorted(xs)
    return xs[min(len(xs) - 1, max(0, math.ceil(q / 100 * len(xs)) - 1))]


def c5_loop(tv, d, rt, N: int, base: str, layers: int, steps: int, train_ms: float,
            inline_gc: bool = False, recycle: bool = True) -> dict:
    """C5 (BASELINE configs[4]): ``Checkpointer(keep_last=3)`` async save EVERY step of a
    synthetic training loop (fixed GPU time + an in-place update of every param shard);
    the blocking time is what the loop spends in ``save_step`` plus the snapshot
    kernel's device time on the training stream (``training_manager.py:191-224``)."""
    import torch

    mesh = tv.Mesh.create([("fsdp", N)], process_count=N)
    leaves = llama_leaves(**dict(LLAMA3_8B, layers=layers))
    tree_bytes = sum(nbytes(s, dt) for _, _, s, dt in leaves)
    # keep_last=3 plus the save in flight live on the storage at once; on a RAM-backed
    # target that must fit host memory, or the kernel OOM-kills the job mid-save
    need, room = 4 * tree_bytes, _storage_room(base)
    if room is not None and need > room:
        raise SystemExit(f"c5: {need / 1e9:.1f} GB of checkpoints (keep_last=3 + 1 in flight) do not fit "
                         f"the {room / 1e9:.1f} GB free on {base}; pass --layers to shrink the tree")
    state, shardings = build_state(tv, rt, mesh, leaves)
    params = [t for p, leaf in tv.flatten(state["state"]["params"]) for t in leaf.shards.values()]
    torch.cuda.synchronize()
    # the synchronous save this replaces
    sync_ms = []
    for i in range(2):
        d.barrier()
        t0 = time.perf_counter()
        tv.save_checkpoint(rt, f"c5sync/{i}", state, shardings, tv.SaveOptions(sync=True)).wait()
        sync_ms.append(d.max((time.perf_counter() - t0) * 1e3))
        d.barrier()
        if d.rank == 0:
            shutil.rmtree(os.path.join(base, "c5sync"), ignore_errors=True)
    sync_save_ms = sync_ms[-1]
    cycles = int(train_ms * 1.965e6)
    ck = tv.Checkpointer(rt, "c5run", tv.RetentionPolicy(keep_last=3), tv.SaveOptions(sync=False),
                         background_delete=not inline_gc, recycle=recycle)
    blocking, waits, joins, gcs, bg, snap_dev = [], [], [], [], [], []
    phase_sums: dict[str, float] = {}
    from paper_2605_23066_b200 import native
    from paper_2605_23066_b200 import timeline as _tlm

    native.kernel_timing_collect()
    native.kernel_timing(True)  # the snapshot kernel's device time, per step
    t_start = time.perf_counter()
    prev = None
    for step in range(steps):
        # synthetic training step: fixed GPU time + an in-place update of every param shard
        torch.cuda._sleep(cycles)
        for t in params:
            t.mul_(0.999)
        torch.cuda.synchronize()
        d.barrier()
        t0 = time.perf_counter()
        handle = ck.save_step(step, state, shardings)
        blocking.append(d.max((time.perf_counter() - t0) * 1e3))
        torch.cuda.synchronize()  # the snapshot kernel queued on the training stream
        kt = native.kernel_timing_collect()
        snap_dev.append(d.max(kt["ms_max"]))
        waits.append(d.max(ck.last_wait_seconds * 1e3))
        joins.append(d.max(ck.last_join_seconds * 1e3))
        gcs.append(d.max(ck.last_gc_seconds * 1e3))
        if prev is not None:  # the previous save has been joined: its per-phase timeline is final
            for k, v in _tlm.LAST_SAVE.get(d.rank if d.on else 0, {}).items():
                phase_sums[k] = phase_sums.get(k, 0.0) + v
            tl = prev.handles[0].session.timeline
            if "finalized" in tl and "snapshotted" in tl:
                bg.append((tl["finalized"] - tl["snapshotted"]) * 1e3)
        prev = handle
    ck.close()
    native.kernel_timing(False)
    native.kernel_timing_collect()
    loop_s = time.perf_counter() - t_start
    kept = ck.all_steps()
    assert kept == list(range(steps - 3, steps)), kept
    snap = [b - w for b, w in zip(blocking, waits)]
    total = [b + s for b, s in zip(blocking, snap_dev)]
    steady = total[1:] or total  # the first save_step also warms plan caches
    host_steady = blocking[1:] or blocking
    mean = statistics.mean(steady)
    # recycling steady state: step k reuses step k-4's files (keep_last=3 + the save in
    # flight), and a file is CUDA-registered the first time its process claims it, so
    # from step 8 every save overwrites registered files
    warm = 2 * (3 + 1)
    recycled = total[warm:]
    del state, params
    d.barrier()
    if d.rank == 0:
        shutil.rmtree(os.path.join(base, "c5run"), ignore_errors=True)
    torch.cuda.empty_cache()
    return {
        "workload": f"C5 Checkpointer(keep_last=3, async) every step over {steps} steps, Llama-3-8B "
                    f"{layers} layers ({tree_bytes} bytes) FSDP-{N}, synthetic training step = {train_ms} ms "
                    f"GPU time + in-place param update, retention deletes "
                    f"{'inline (reference)' if inline_gc else 'in the background'}",
        "tree_bytes": tree_bytes,
        "blocking_ms_mean": round(mean, 2),
        "blocking_ms_p50": round(_pct(steady, 50), 2),
        "blocking_ms_p99": round(_pct(steady, 99), 2),
        "blocking_ms_max": round(max(steady), 2),
        "blocking_host_ms_mean": round(statistics.mean(host_steady), 2),
        "snapshot_device_ms_mean": round(statistics.mean(snap_dev[1:] or snap_dev), 2),
        "wait_on_previous_ms_mean": round(statistics.mean(waits[1:] or waits), 2),
        "own_sync_phase_ms_mean": round(statistics.mean(snap[1:] or snap), 2),
        "join_previous_ms_mean": round(statistics.mean(joins[1:] or joins), 2),
        "retention_gc_ms_mean": round(statistics.mean(gcs[1:] or gcs), 2),
        "background_save_ms_mean": round(statistics.mean(bg), 2) if bg else None,
        "sync_save_ms": round(sync_save_ms, 2),
        "blocking_frac_of_sync_save": round(mean / sync_save_ms, 4),
        "blocking_p99_frac_of_sync_save": round(_pct(steady, 99) / sync_save_ms, 4),
        "steady_state": ({"from_step": warm, "blocking_ms_mean": round(statistics.mean(recycled), 2),
                          "blocking_ms_p99": round(_pct(recycled, 99), 2),
                          "frac_of_sync_save": round(statistics.mean(recycled) / sync_save_ms, 4),
                          "note": "steps whose save overwrites recycled, already-registered files"}
                         if recycled else None),
        "loop_seconds": round(loop_s, 2),
        "retained_steps": kept,
        "blocking_ms_per_step": [round(x, 2) for x in total],
        "background_save_ms_per_step": [round(x, 1) for x in bg],
        "save_phases_ms_mean_rank0": {k: round(v / max(1, steps - 1), 2) for k, v in phase_sums.items()},
        "how": "blocking per step = wall time in save_step (max over ranks) + the snapshot kernel's device "
               "time on the training stream (CUDA events, libtvgpu tv_kernel_timing); first step excluded",
    }


def run_c5(args) -> dict:
    """C5 as the whole bench line (``--config c5``)."""
    import torch

    import paper_2605_23066_b200 as tv

    d = Dist()
    d.init()
    N = d.world if d.on else args.gpus
    torch.cuda.set_device(d.local)
    base = args.dir
    if d.rank == 0:
        shutil.rmtree(base, ignore_errors=True)
        os.makedirs(base, exist_ok=True)
    d.barrier()
    backend = tv.FilesystemBackend(base)
    rt = open_runtime(tv, d, N, backend, gpus=list(range(N)))
    res = c5_loop(tv, d, rt, N, base, args.layers, args.steps, args.train_ms, args.inline_gc, args.recycle)
    d.barrier()
    if d.rank == 0:
        shutil.rmtree(base, ignore_errors=True)
    return {
        "metric": "async-save blocking time per training step (Checkpointer.save_step every step)",
        "value": res["blocking_ms_mean"],
        "unit": "ms",
        "higher_is_better": False,
        "n_gpus": N,
        "steps": args.steps,
        "config": {"workload": res["workload"], "config": "c5"},
        **{k: v for k, v in res.items() if k != "workload"},
    }


def time_launch(fn, gpu: int, reps: int = 5, warmup: int = 3) -> tuple[float, float]:
    """(median kernel ms by CUDA events on the launching stream, median host enqueue ms).
    The stream is held by a short device-side sleep while the host enqueues, so the event
    window contains the kernel only."""
    import torch

    with torch.cuda.device(gpu):
        stream = torch.cuda.current_stream(gpu)
        for _ in range(warmup):
            fn(stream)
        torch.cuda.synchronize(gpu)
        dev_ms, host_ms = [], []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(20_000_000)  # ~10 ms of GPU time covers the host enqueue
            a.record(stream)
            t0 = time.perf_counter()
            fn(stream)
            host_ms.append((time.perf_counter() - t0) * 1e3)
            b.record(stream)
            b.synchronize()
            dev_ms.append(a.elapsed_time(b))
    return statistics.median(dev_ms), statistics.median(host_ms)


def _ncu_traffic(bytes_per_launch: int):
    """DRAM bytes per launch of the same kernel launch from a committed ncu capture
    (dram__bytes_read.sum + dram__bytes_write.sum; the current build's capture first,
    profiles/r02_roofline_traffic_full.json, then round 1's), used only when that
    capture's launch moved exactly the bytes this one did."""
    for name in ("r02_roofline_traffic_full.json", "r01_roofline_traffic.json"):
        path = os.path.join(ROOT, "profiles", name)
        if not os.path.exists(path):
            continue
        with open(path) as f:
            rows = json.load(f).get("launches", [])
        for r in rows:
            if int(r["algorithmic_bytes"]) == int(bytes_per_launch):
                return int(r["dram_read_bytes"]) + int(r["dram_write_bytes"]), f"{r.get('source')} [{name}]"
    return None, None


def kernel_roofline(tv, native, state, rt, d, ksave: dict, kload: dict, args, step_ms: float,
                    peer_gb: float = 0.0) -> dict:
    """The box-copy kernel inside the timed steps, timed live by libtvgpu with CUDA events on
    the launching stream (tv_kernel_timing); algorithmic bytes = 2 × bytes copied.  Save side
    (async mode): the device snapshot, ONE launch per GPU per step.  Restore side: unpack /
    reshard fan-out launches (none when every chunk lands contiguously by DMA).  The
    dominant one (more device time) is reported, the other beside it.  With no kernel in
    the timed region (sync mode, aligned restore) the snapshot launch is timed standalone
    and marked launches_in_timed_region = 0."""
    import torch

    peak = measured_peaks()["hbm_gbs"]
    world = d.world if d.on else 1

    def summary(k, name):
        launches = int(d.sum(k["launches"]))
        if launches == 0:
            return None
        ms_total = d.sum(k["ms_total"])
        nbytes = d.sum(k["bytes"])
        per_launch = int(round(nbytes / launches))
        achieved = nbytes / (ms_total / 1e3) / 1e9
        traffic, src = _ncu_traffic(per_launch)
        return {
            "kernel": name,
            "bound": "hbm",
            "achieved": round(achieved, 1),
            "peak": peak,
            "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "traffic": traffic,
            "traffic_source": src,
            "bytes_per_launch": per_launch,
            "ms_per_launch": round(ms_total / launches, 3),
            "ms_max_launch": round(d.max(k["ms_max"]), 3),
            "launches_in_timed_region": launches,
            "share_of_step": round(ms_total / world / args.steps / step_ms, 5),
            "timing": "CUDA events on the launching stream around every launch in the timed steps "
                      "(libtvgpu tv_kernel_timing), summed over ranks",
        }

    s_sum = summary(ksave, "box_copy_kernel (async-save device snapshot: this GPU's write ranges -> "
                           "arena, 1 launch per GPU per step)")
    l_sum = summary(kload, "box_copy_kernel (restore unpack / reshard fan-out into local and peer HBM)")
    if l_sum is not None and peer_gb > 0:
        # the fan-out's binding link: bytes stored into peer HBM leave each GPU over NVLink;
        # per-GPU egress = peer bytes / (summed kernel time / GPUs), against the measured
        # 770 GB/s peer-copy bandwidth per direction (B200_PROFILING.md)
        n_gpus = d.world if d.on else max(1, args.restore_gpus or args.gpus)
        per_gpu_s = d.sum(kload["ms_total"]) / 1e3 / n_gpus
        nv = peer_gb / per_gpu_s / n_gpus
        l_sum["nvlink"] = {"peer_GB_in_timed_steps": round(peer_gb, 3),
                           "achieved_GBps_per_gpu": round(nv, 1), "peak_GBps_per_gpu": 770.0,
                           "frac": round(nv / 770.0, 4),
                           "peak_source": "B200_PROFILING.md measured peer copy, per direction"}
    live = [x for x in (s_sum, l_sum) if x is not None]
    if live:
        best = max(live, key=lambda x: x["ms_per_launch"] * x["launches_in_timed_region"])
        other = [x for x in live if x is not best]
        if other:
            best = dict(best, other_kernel_in_step=other[0])
        return best

    regions = []
    for tree in state.values():
        for path, leaf in tv.flatten(tree):
            for dev, t in _device_tensors(leaf):
                regions.append(t)
    gpu = regions[0].device.index
    regions = [t for t in regions if t.device.index == gpu]
    total = sum(t.numel() * t.element_size() for t in regions)
    offs, cur = [], 0
    for t in regions:
        offs.append(cur)
        cur += (t.numel() * t.element_size() + 255) & ~255
    arena = torch.empty(cur, dtype=torch.uint8, device=f"cuda:{gpu}")
    base = arena.data_ptr()
    copies = native.copy_table(
        [t.data_ptr() for t in regions], [tuple(t.shape) for t in regions],
        [(0,) * t.dim() for t in regions], [base + o for o in offs], [tuple(t.shape) for t in regions],
        [(0,) * t.dim() for t in regions], [tuple(t.shape) for t in regions],
        [t.element_size() for t in regions],
    )
    ms, host_ms = time_launch(lambda s: native.copy_boxes(gpu, copies, s.cuda_stream), gpu)
    achieved = 2 * total / (ms / 1e3) / 1e9
    del arena
    traffic, src = _ncu_traffic(2 * total)
    return {
        "kernel": "box_copy_kernel (device snapshot: all local shards -> arena, 1 launch, standalone)",
        "bound": "hbm",
        "achieved": round(achieved, 1),
        "peak": peak,
        "unit": "GB/s",
        "frac": round(achieved / peak, 4),
        "traffic": traffic,
        "traffic_source": src,
        "bytes_per_launch": 2 * total,
        "ms_per_launch": round(ms, 3),
        "host_enqueue_ms": round(host_ms, 3),
        "launches_in_timed_region": 0,
    }


def retire_checkpoint(d, backend, path: str, recycle: bool) -> None:
    """Retire a checkpoint as retention would (``training_manager.delete_checkpoint``:
    finality marker first, then everything else), the bulk spread over the ranks: under
    torchrun process 0 removes the marker, then every rank its own ``process_<p>/`` files
    in parallel, then process 0 the remaining top-level documents."""
    from paper_2605_23066_b200.training_manager import _finality_marker, delete_checkpoint

    store = backend.store("retention")
    if not d.on:
        delete_checkpoint(store, path, recycle=recycle)
        return
    if d.rank == 0:
        marker = f"{path}/{_finality_marker(store)}"
        if store.exists(marker):
            store.delete(marker)
    d.barrier()
    delete_checkpoint(store, f"{path}/process_{d.rank}", recycle=recycle)
    d.barrier()
    if d.rank == 0:
        delete_checkpoint(store, path, recycle=recycle)


def c3_leg(tv, native, d, rt, backend, args, N: int, base: str) -> dict:
    """BASELINE configs[2] in the default line at N >= 4 (N = 8 is its 2 x 4 mesh, P = 8):
    the same tree on a (replica 2 x fsdp N/2) mesh, replica-parallel save (each replica
    GPU writes 1/2 of its shard) + restore onto the same mesh, the step's save mode,
    recycled + registered files like the main loop.  Timed like the step (CUDA events,
    barrier + sync, max over ranks); the last restore is verified on the device."""
    import dataclasses

    import torch

    leaves = llama_leaves(**dict(LLAMA3_8B, layers=args.layers))
    tree_bytes = sum(nbytes(s, dt) for _, _, s, dt in leaves)
    mesh = tv.Mesh.create([("replica", 2), ("fsdp", N // 2)], process_count=N, replica_axis="replica")
    target = f"2x{N // 2} (replica x fsdp), {N} processes, replica-parallel save"
    # state + restored copy (+ the async snapshot arena) per GPU, each 2 x tree / N
    per_gpu = 2 * tree_bytes // N * (3 if args.save_mode == "async" else 2)
    dev = d.local if d.on else 0
    free = torch.cuda.mem_get_info(dev)[0] + torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
    if d.max(-free) > -(per_gpu + (4 << 30)):
        return {"target": target, "skipped": f"needs {per_gpu / 1e9:.1f} GB of free HBM per GPU"}
    state, shardings = build_state(tv, rt, mesh, leaves, seed=3, spec_fn=fsdp_spec)
    opts = tv.SaveOptions(sync=args.save_mode == "sync", replica_parallel=True, layout=args.layout)
    backend.register_pool = bool(args.recycle) and not args.no_register
    saves, restores, verified = [], [], {}
    warm = 3
    for i in range(warm + args.c3_steps):
        path = f"bench/c3_{i}"
        d.barrier()
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        tv.save_checkpoint(rt, path, state, shardings, opts).wait()
        e1.record()
        out = tv.load_checkpoint(rt, path, None, tv.LoadOptions(), current_mesh=mesh)
        e2.record()
        torch.cuda.synchronize()
        if i >= warm:
            saves.append(d.max(e0.elapsed_time(e1)))
            restores.append(d.max(e1.elapsed_time(e2)))
        if i == warm + args.c3_steps - 1:
            nb, bad = verify_restore(tv, state, out, leaves, seed=3)
            verified = {"bytes_compared": int(d.sum(nb)), "mismatched_boxes": int(d.sum(bad))}
        del out
        d.barrier()
        retire_checkpoint(d, backend, path, args.recycle)
        if d.rank == 0:
            shutil.rmtree(os.path.join(base, path), ignore_errors=True)
        d.barrier()
    del state
    backend.register_pool = False
    free_recycle_pool(native, d, backend)
    torch.cuda.empty_cache()
    save_ms, restore_ms = statistics.mean(saves), statistics.mean(restores)
    return {
        "target": target,
        "GBps": round(2 * tree_bytes / ((save_ms + restore_ms) / 1e3) / 1e9, 3),
        "save_GBps": round(tree_bytes / (save_ms / 1e3) / 1e9, 3),
        "restore_GBps": round(tree_bytes / (restore_ms / 1e3) / 1e9, 3),
        "save_ms": round(save_ms, 2),
        "restore_ms": round(restore_ms, 2),
        "steps": args.c3_steps,
        "warmup": warm,
        "tree_bytes": tree_bytes,
        "restore_verified": dict(verified, how="every restored shard (both replicas) against the saved "
                                               "state, torch.equal on the device (all ranks)"),
        "note": "GB/s counts the tree once per save and once per restore (as the metric); the "
                "restore lands 2 x tree bytes in HBM (both replicas; stored chunks read once, "
                "fanned out over NVLink)",
    }


def c1_leg(tv, native, d, base: str, args) -> dict | None:
    """BASELINE configs[0] in the default line: a single-process save + restore round trip
    of 4 x (4096, 4096) f32 unsharded arrays (268 MB) to the same storage, on process 0's
    GPU (rank 0 only under torchrun), timed per step like the main step (async save +
    wait + restore + retire), restored bytes verified."""
    import torch

    from paper_2605_23066_b200.training_manager import delete_checkpoint

    d.barrier()
    if d.rank != 0:
        d.barrier()
        return None
    gpu = d.local if d.on else 0
    sub = os.path.join(base, "c1leg")
    backend = tv.FilesystemBackend(sub, register_pool=bool(args.recycle) and not args.no_register)
    rt = tv.SimulatedRuntime(1, backend, gpus=[gpu])
    gen = torch.Generator(device=f"cuda:{gpu}")
    gen.manual_seed(0)
    arrays = {f"a{i}": torch.empty((4096, 4096), dtype=torch.float32, device=f"cuda:{gpu}").normal_(generator=gen)
              for i in range(4)}
    tree = {"model": {k: tv.DenseArray("f32", v) for k, v in arrays.items()}}
    nbytes = 4 * 4096 * 4096 * 4
    times, saves, restores = [], [], []
    bad = 0
    for i in range(args.c1_warmup + args.c1_steps):
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        tv.save_checkpoint(rt, f"c1/{i}", tree, None, tv.SaveOptions(sync=args.save_mode == "sync")).wait()
        e1.record()
        out = tv.load_checkpoint(rt, f"c1/{i}", None, tv.LoadOptions())
        e2.record()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        delete_checkpoint(backend.store("retention"), f"c1/{i}", recycle=args.recycle)
        retire = (time.perf_counter() - t0) * 1e3
        if i == args.c1_warmup + args.c1_steps - 1:
            bad = sum(0 if torch.equal(out["model"][k].data.view(torch.int32), v.view(torch.int32)) else 1
                      for k, v in arrays.items())
        del out
        if i >= args.c1_warmup:
            saves.append(e0.elapsed_time(e1))
            restores.append(e1.elapsed_time(e2))
            times.append(e0.elapsed_time(e2) + retire)
    backend.drain_recycle_pool()
    shutil.rmtree(sub, ignore_errors=True)
    d.barrier()
    ms = statistics.mean(times)
    return {
        "workload": "C1 4 x (4096,4096) f32 unsharded (268435456 bytes), one process, "
                    f"{args.save_mode} save + restore + retire per step",
        "value": round(2 * nbytes / (ms / 1e3) / 1e9, 3),
        "unit": "GB/s",
        "ms_per_step": round(ms, 2),
        "save_GBps": round(nbytes / (statistics.mean(saves) / 1e3) / 1e9, 3),
        "restore_GBps": round(nbytes / (statistics.mean(restores) / 1e3) / 1e9, 3),
        "steps": args.c1_steps,
        "warmup": args.c1_warmup,
        "restore_verified": {"bytes_compared": nbytes, "mismatched_arrays": bad},
    }


def free_recycle_pool(native, d, backend) -> None:
    """Between bench legs: free the recycle pool (process 0) and every rank's CUDA
    registrations of its files, so the next leg's tree has the RAM-backed storage."""
    d.barrier()
    if d.rank == 0:
        backend.drain_recycle_pool()
    d.barrier()
    native.lib().tv_mapping_release_all()
    d.barrier()


def reshard_leg(tv, native, d, rt, wl, state, shardings, args, N: int, base: str) -> dict:
    """BASELINE's reshard GB/s in the default line: the step's checkpoint (FSDP-N) restored
    onto another sharding of the same GPUs — at N >= 2 the C4 target shape (replica 2 x
    fsdp N/2: every stored chunk is consumed by two GPUs, read once, fanned out over
    NVLink by the unpack kernel); at N = 1 a column split (None, "tp") over 2 logical
    devices (every byte through the unpack kernel).  Timed like the step (CUDA events,
    barrier + sync, max over ranks); the last restore is verified on the device."""
    import torch

    if N >= 2:
        mesh = tv.Mesh.create([("replica", 2), ("fsdp", N // 2)], process_count=N, replica_axis="replica")
        spec_fn, target = fsdp_spec, f"2x{N // 2} (replica x fsdp), {N} processes"
        rrt = rt
    else:
        mesh = tv.Mesh.create([("tp", 2)], process_count=2)
        spec_fn = lambda s: (None, "tp") if len(s) == 2 else ("tp",)  # noqa: E731
        target, rrt = "(None, 'tp') column split over 2 logical devices on GPU 0", \
            tv.SimulatedRuntime(2, rt.backend, gpus=[0])
    tree: dict = {}
    for t, path, shape, dtype in wl.leaves:
        node = tree.setdefault(t, {})
        parts = path.split("/")
        for p in parts[:-1]:
            node = node.setdefault(p, {})
        node[parts[-1]] = tv.AbstractLeaf("array", shape, dtype,
                                          tv.Sharding(mesh, tv.PartitionSpec(spec_fn(shape)), shape))
    abstract = {"state": tree}
    # the restored copy lives next to the state: skip (with a note) when HBM cannot hold it
    per_gpu = wl.tree_bytes * (2 if N >= 2 else 1) // max(1, N)
    dev = d.local if d.on else 0
    # free HBM plus blocks the caching allocator holds but nothing uses (e.g. the async
    # snapshot arena of the last save, cached on the caller's stream)
    free = torch.cuda.mem_get_info(dev)[0] + torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
    if d.max(-free) > -(per_gpu + (4 << 30)):  # min over ranks of free HBM < need
        return {"target": target, "skipped": f"needs {per_gpu / 1e9:.1f} GB of free HBM per GPU next to the "
                                             f"state; have {d.max(-free) * -1 / 1e9:.1f}"}
    path = "bench/reshard"
    tv.save_checkpoint(rt, path, state, shardings, tv.SaveOptions(sync=True)).wait()
    times, nv = [], []
    verified = {}
    for i in range(args.reshard_steps):
        before = native.totals()["peer_bytes"]
        d.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = tv.load_checkpoint(rrt, path, abstract, tv.LoadOptions())
        e1.record()
        torch.cuda.synchronize()
        times.append(d.max(e0.elapsed_time(e1)))
        nv.append(d.sum(native.totals()["peer_bytes"] - before))
        if i == args.reshard_steps - 1:
            nb, bad = verify_restore(tv, state, out, wl.leaves)
            verified = {"bytes_compared": int(d.sum(nb)), "mismatched_boxes": int(d.sum(bad))}
        del out  # (no empty_cache: the next restore reuses the block, peers' mappings stay valid)
    d.barrier()
    if d.rank == 0:
        from paper_2605_23066_b200.training_manager import delete_checkpoint

        delete_checkpoint(rt.backend.store("retention"), path, recycle=args.recycle)
        shutil.rmtree(os.path.join(base, "bench"), ignore_errors=True)
    ms = statistics.mean(times)
    return {
        "target": target,
        "GBps": round(wl.tree_bytes / (ms / 1e3) / 1e9, 3),
        "ms": round(ms, 2),
        "restores": args.reshard_steps,
        "nvlink_GB_per_restore": round(statistics.mean(nv) / 1e9, 3),
        "restore_verified": dict(verified, how="every restored shard's overlap with every saved shard, "
                                               "torch.equal on the device (all ranks)"),
    }


def verify_restore(tv, state, out, leaves=None, seed: int = 0) -> tuple[int, int]:
    """Restored shards vs the saved state, byte for byte on the device: each target shard's
    overlap with EVERY source shard must be equal (any target sharding).  Source shards
    this process does not hold (torchrun: other ranks' shards) are regenerated on the
    target's GPU with ``gen_shard`` when ``leaves`` (the workload's leaf list) is given.
    Returns (bytes compared, mismatching boxes)."""
    import torch

    index = {f"{t}/{p}": (i, t, dt) for i, (t, p, _, dt) in enumerate(leaves)} if leaves else {}
    ints = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}
    compared = bad = 0
    for name, tree in out.items():
        src = dict(tv.flatten(state[name]))
        for path, leaf in tv.flatten(tree):
            ref = src[path]
            if not hasattr(leaf, "shards") or not hasattr(ref, "shards"):
                if hasattr(leaf, "data") and hasattr(ref, "data") and hasattr(leaf.data, "is_cuda"):
                    a, b = leaf.data, ref.data.to(leaf.data.device)  # unsharded (C1): whole arrays
                    a, b = a.view(ints[a.element_size()]), b.view(ints[b.element_size()])
                    compared += a.numel() * a.element_size()
                    bad += 0 if torch.equal(a, b) else 1
                continue
            t_ranges = leaf.shard_ranges()
            ref_ranges = ref.shard_ranges()
            source_boxes = {}
            for sh in tv.shards_of(ref.sharding):
                source_boxes.setdefault(sh.ranges, sh.device)  # one replica per range
            for tdev, t in leaf.shards.items():
                tr = t_ranges[tdev]
                for sr, sdev in source_boxes.items():
                    hit = []
                    for (a0, ae), (b0, be) in zip(tr, sr):
                        lo, hi = max(a0, b0), min(a0 + ae, b0 + be)
                        if hi <= lo:
                            hit = None
                            break
                        hit.append((lo, hi - lo))
                    if hit is None:
                        continue
                    sv = ref.shards.get(sdev)
                    if sv is None:  # held by an equal-range replica here, or regenerate
                        sv = next((ref.shards[d] for d, r in ref_ranges.items()
                                   if r == sr and d in ref.shards), None)
                    if sv is None:
                        if path not in index:
                            continue
                        i, tname, dt = index[path]
                        sv = gen_shard(i, tname, dt, sr, seed, t.device.index)
                    a = t[tuple(slice(o - to, o - to + e) for (o, e), (to, _) in zip(hit, tr))]
                    b = sv[tuple(slice(o - so, o - so + e) for (o, e), (so, _) in zip(hit, sr))]
                    if b.device != a.device:
                        b = b.to(a.device)
                    a, b = a.view(ints[a.element_size()]), b.view(ints[b.element_size()])
                    compared += a.numel() * a.element_size()
                    bad += 0 if torch.equal(a, b) else 1  # bit patterns (NaN-safe)
    return compared, bad


def _device_tensors(leaf):
    return leaf.shards.items() if hasattr(leaf, "shards") else [(-1, leaf.data)]


def end_to_end(tv, rt, wl, args, d, base) -> dict:
    """Same metric through the public API with HOST buffers, on the same bounded sample
    the reference arm times (``sample_leaves``): per step the inputs go H2D from pinned
    host memory, then ``save_checkpoint`` (the step's save mode) + ``wait()`` +
    ``load_checkpoint``, then the restored shards go D2H into pinned host memory — all
    inside the timed region.  Mesh: our arm's (one logical process per GPU)."""
    import dataclasses

    import torch

    mesh = wl.save_mesh
    e_leaves = sample_leaves(wl.name, args.cpu_layers)
    opts = dataclasses.replace(wl.save_options, sync=args.save_mode == "sync")
    # host copies of this process's shards (pinned), generated from the device state
    state, shardings = build_state(tv, rt, mesh, e_leaves, seed=7, spec_fn=wl.spec_fn)
    host = {}
    local_bytes = 0
    for tree in state.values():
        for path, leaf in tv.flatten(tree):
            for dev, t in _device_tensors(leaf):
                h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                h.copy_(t)
                host[(path, dev)] = h
                local_bytes += t.numel() * t.element_size()
    torch.cuda.synchronize()
    tree_bytes = sum(nbytes(s, dt) for _, _, s, dt in e_leaves)
    times = []
    for i in range(args.e2e_warmup + args.e2e_steps):
        d.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for tree in state.values():  # H2D: inputs from pinned host memory
            for path, leaf in tv.flatten(tree):
                for dev, t in _device_tensors(leaf):
                    t.copy_(host[(path, dev)], non_blocking=True)
        torch.cuda.synchronize()
        path = f"e2e/step_{i}"
        tv.save_checkpoint(rt, path, state, shardings, opts).wait()
        out = tv.load_checkpoint(rt, path, None, tv.LoadOptions(), current_mesh=mesh)
        for tree in out.values():  # D2H: restored shards to pinned host memory
            for p, leaf in tv.flatten(tree):
                for dev, t in _device_tensors(leaf):
                    host[(p, dev)].copy_(t, non_blocking=True)
        torch.cuda.synchronize()
        del out
        d.barrier()
        if d.rank == 0:  # retire it, as the main step does
            from paper_2605_23066_b200.training_manager import delete_checkpoint

            delete_checkpoint(rt.backend.store("retention"), path, recycle=args.recycle)
        dt = d.max(time.perf_counter() - t0)
        d.barrier()
        if i >= args.e2e_warmup:
            times.append(dt)
    del state, host
    torch.cuda.empty_cache()
    sec = statistics.mean(times)
    total_local = d.sum(local_bytes)
    return {
        "value": round(2 * tree_bytes / sec / 1e9, 3),
        "unit": "GB/s",
        "h2d_bytes_per_step": int(total_local),
        "d2h_bytes_per_step": int(total_local),
        "tree_bytes": tree_bytes,
        "sample": (f"the reference arm's sample: {len(e_leaves)} leaves"
                   + ("" if wl.name == "c1" else f" ({args.cpu_layers} layers + final_norm, no embed/lm_head)")),
        "config": wl.name,
        "api": f"save_checkpoint({args.save_mode}) + wait() + load_checkpoint + retire, with H2D of the "
               "inputs and D2H of the restored shards (pinned) inside the timed region",
        "steps": args.e2e_steps,
        "warmup": args.e2e_warmup,
    }


# -- the reference arm / CPU baseline -----------------------------------------------------------


def sample_leaves(config: str, layers: int):
    """The bounded sample both CPU legs and our e2e run: the whole C1 tree for c1; else
    ``layers`` transformer layers of the C2 tree plus final_norm (no embed / lm_head)."""
    if config == "c1":
        return [("model", f"a{i}", (4096, 4096), "f32") for i in range(4)]
    return [(t, p, s, dt) for t, p, s, dt in llama_leaves(**dict(LLAMA3_8B, layers=layers))
            if not p.startswith(("embed", "lm_head"))]


def reference_processes(config: str) -> int:
    """Simulated processes of the reference's multi-controller mode (one host thread
    each): every host thread it can use (a power of two), 1 for C1 (unsharded)."""
    if config == "c1":
        return 1
    cores = len(os.sched_getaffinity(0))
    return max(1, min(64, 1 << (cores.bit_length() - 1)))


def _host_tree(leaves, seed=0):
    import numpy as np

    rng = np.random.default_rng(seed)
    tree: dict = {}
    for t, p, shape, dt in leaves:
        node = tree.setdefault(t, {})
        parts = p.split("/")
        for q in parts[:-1]:
            node = node.setdefault(q, {})
        if dt == "bf16":
            data = rng.integers(0, 1 << 16, size=shape, dtype=np.uint16)
        else:
            data = rng.standard_normal(size=shape, dtype=np.float32)
        node[parts[-1]] = data
    return tree


def reference_leg(args, root_dir: str, steps: int, warmup: int) -> dict:
    """The UNMODIFIED reference (oracle/_ref, staged by oracle/ref_recipe.py from
    /root/reference/pkg/src/treevault) through its own public API: per step an async
    ``save_checkpoint(...).wait()`` (``save_pipeline.py:594-622``) and a
    ``load_checkpoint`` of it (``load_pipeline.py:538-580``) on the same storage target as
    our arm, P simulated processes (one host thread each), FSDP-P on dim 0."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref_recipe

    rv = ref_recipe.load_reference()
    config = getattr(args, "config", "c2")
    leaves = sample_leaves(config, args.cpu_layers)
    P = reference_processes(config)
    host = _host_tree(leaves)
    mesh = rv.Mesh.create([("fsdp", P)], process_count=P)
    tree, shardings = {}, {}
    for t, p, shape, dt in leaves:
        node, src = tree.setdefault(t, {}), host[t]
        parts = p.split("/")
        for q in parts[:-1]:
            node, src = node.setdefault(q, {}), src[q]
        node[parts[-1]] = rv.DenseArray(dt, src[parts[-1]])
        if config != "c1":
            shardings[f"{t}/{p}"] = rv.Sharding(mesh, rv.PartitionSpec(("fsdp",) + (None,) * (len(shape) - 1)), shape)
    sample_bytes = sum(nbytes(s, dt) for _, _, s, dt in leaves)
    root = os.path.join(root_dir, "reference_arm")
    saves, restores = [], []
    for i in range(warmup + steps):
        shutil.rmtree(root, ignore_errors=True)
        os.makedirs(root)
        rt = rv.SimulatedRuntime(P, rv.FilesystemBackend(root))
        t0 = time.perf_counter()
        rv.save_checkpoint(rt, "ck", {"state": tree}, {"state": shardings} if shardings else None,
                           rv.SaveOptions(sync=False)).wait()
        t1 = time.perf_counter()
        out = rv.load_checkpoint(rt, "ck", None, rv.LoadOptions(), current_mesh=mesh if shardings else None)
        t2 = time.perf_counter()
        del out
        if i >= warmup:
            saves.append(t1 - t0)
            restores.append(t2 - t1)
    shutil.rmtree(root, ignore_errors=True)
    t_save, t_restore = statistics.mean(saves), statistics.mean(restores)
    return {
        "value": round(2 * sample_bytes / (t_save + t_restore) / 1e9, 3),
        "unit": "GB/s",
        "cores": P,
        "kind": "reference",
        "sample": (f"the whole C1 tree (4 x (4096,4096) f32, unsharded, one process), {sample_bytes} bytes"
                   if config == "c1" else
                   f"{args.cpu_layers} transformer layers of the C2 tree + final_norm (no embed/lm_head), "
                   f"{sample_bytes} bytes, FSDP-{P} over {P} simulated processes (one host thread each)")
                  + f"; async save().wait() + load_checkpoint per step, mean of {steps} after {warmup} warm-up",
        "sample_bytes": sample_bytes,
        "save_GBps": round(sample_bytes / t_save / 1e9, 3),
        "restore_GBps": round(sample_bytes / t_restore / 1e9, 3),
        "implementation": "treevault (unmodified, oracle/_ref) via save_checkpoint / load_checkpoint",
    }


def port_leg(args, root_dir: str, steps: int = 1, warmup: int = 0) -> dict:
    """Cross-check: the oracle port (oracle/treevault_oracle.py restating save_pipeline /
    chunkstore / load_pipeline) on the same sample and process count."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import treevault_oracle as orc

    config = getattr(args, "config", "c2")
    leaves = sample_leaves(config, args.cpu_layers)
    P = reference_processes(config)
    host = _host_tree(leaves)
    tree: dict = {"state": {}}
    specs: dict = {"state": {}}
    for t, p, shape, dt in leaves:
        node, src = tree["state"].setdefault(t, {}), host[t]
        parts = p.split("/")
        for q in parts[:-1]:
            node, src = node.setdefault(q, {}), src[q]
        node[parts[-1]] = ("array", dt, src[parts[-1]])
        if config != "c1":
            specs["state"][f"{t}/{p}"] = ([("fsdp", P)], P, None, ("fsdp",) + (None,) * (len(shape) - 1))
    sample_bytes = sum(nbytes(s, dt) for _, _, s, dt in leaves)
    root = os.path.join(root_dir, "port_leg")
    saves, restores = [], []
    for i in range(warmup + steps):
        shutil.rmtree(root, ignore_errors=True)
        os.makedirs(root)
        t0 = time.perf_counter()
        files = orc.expected_checkpoint(tree, specs, {}, P, "fs", path="ck")
        keys = sorted(files)
        per = [dict((k, files[k]) for k in keys[j::P]) for j in range(P)]
        ths = [threading.Thread(target=orc.save_to_directory, args=(root, part)) for part in per]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        t_save = time.perf_counter() - t0
        del files, per
        t0 = time.perf_counter()
        restored = orc.restore_from_directory(root, "ck", P)
        t_restore = time.perf_counter() - t0
        del restored
        if i >= warmup:
            saves.append(t_save)
            restores.append(t_restore)
    shutil.rmtree(root, ignore_errors=True)
    t_save, t_restore = statistics.mean(saves), statistics.mean(restores)
    return {"value": round(2 * sample_bytes / (t_save + t_restore) / 1e9, 3), "unit": "GB/s", "cores": P,
            "kind": "port", "sample_bytes": sample_bytes, "steps": steps, "warmup": warmup}


def cpu_baseline(args, root_dir: str) -> dict:
    """``cpu_baseline`` of our line (rank 0, N=1): the reference leg on a bounded sample
    (one warm-up + one timed step), with the port beside it as a cross-check."""
    res = reference_leg(args, root_dir, steps=1, warmup=1)
    try:
        res["port_cross_check"] = port_leg(args, root_dir)
    except Exception as exc:  # noqa: BLE001 - a cross-check must not sink the bench line
        res["port_cross_check"] = {"error": repr(exc)}
    return res


def run_reference(args) -> dict:
    """The reference arm: the unmodified reference on the box's host cores, --warmup W +
    --steps K save+restore steps of a bounded sample of OUR arm's workload (same
    ``config`` object, same storage target), rank 0 only."""
    d = Dist()
    base = prepare_storage(args, d)
    os.makedirs(base, exist_ok=True)
    res = reference_leg(args, base, steps=args.steps, warmup=args.warmup)
    N = d.world if d.on else args.gpus
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": res["value"],
        "unit": "GB/s",
        "n_gpus": N,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u8",
        "payload_dtypes": "bf16 params (as <u2 bit patterns: the reference has no bf16) + f32 Adam mu/nu, "
                          "moved as bytes (no arithmetic on the path)",
        "data": "synthetic (numpy RNG, Llama-3-8B shapes)",
        "config": bench_config(args, N),
        "save_GBps": res["save_GBps"],
        "restore_GBps": res["restore_GBps"],
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample", "implementation")},
        "e2e": {"value": res["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "tree_bytes": res["sample_bytes"]},
    }


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-warmup", type=int, default=3)
    ap.add_argument("--cpu-layers", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dir", default="/dev/shm/tvbench")
    ap.add_argument("--storage", default="hugetmpfs", choices=["shm", "hugetmpfs"],
                    help="hugetmpfs (default; falls back to /dev/shm if it cannot be mounted) or shm")
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c3ss", "c4", "c5"])
    ap.add_argument("--restore-gpus", type=int, default=None)
    ap.add_argument("--layout", default="per_leaf", choices=["per_leaf", "aggregated"],
                    help="per_leaf (one file per chunk, default) or aggregated (64 MiB data files + manifest)")
    ap.add_argument("--save-mode", default="async", choices=["async", "sync"],
                    help="async (default): each step's save is an async save + wait; sync: sync save")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-recycle", dest="recycle", action="store_false",
                    help="retire each step's checkpoint by freeing its files instead of recycling them")
    ap.add_argument("--no-register", action="store_true",
                    help="recycle without registering files with CUDA (no zero-copy; slot ring + pwrite)")
    ap.add_argument("--runtime", default="torchrun", choices=["torchrun", "threads"],
                    help="--gpus N > 1 without torchrun: re-exec under torchrun (default, the driver's "
                         "launch) or run N logical processes as threads of one process")
    ap.add_argument("--train-ms", type=float, default=1000.0)
    ap.add_argument("--c5-layers", type=int, default=8,
                    help="default line: Llama depth of the embedded C5 Checkpointer loop (0 = skip)")
    ap.add_argument("--c5-steps", type=int, default=20)
    ap.add_argument("--c3-steps", type=int, default=3,
                    help="C3 leg of the default line at N >= 4 (replica 2 x fsdp N/2, replica-parallel "
                         "save + restore; 0 = skip)")
    ap.add_argument("--c1-steps", type=int, default=10,
                    help="default line: C1 (4 x 64 MiB f32, one process) round trips after the C2 legs (0 = skip)")
    ap.add_argument("--c1-warmup", type=int, default=3)
    ap.add_argument("--reshard-steps", type=int, default=3,
                    help="default line: restores onto another sharding after the timed steps (0 = skip)")
    ap.add_argument("--inline-gc", action="store_true", help="c5: retention deletes inside wait() (reference)")
    args = ap.parse_args()
    if (args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ
            and args.runtime == "torchrun"):
        # one process per GPU, exactly as the driver launches N > 1: re-exec under torchrun
        import socket

        with socket.socket() as sock:
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    if args.impl == "reference":
        d = Dist()
        if d.on and d.rank != 0:
            return
        print(json.dumps(run_reference(args)))
        return
    result = run_c5(args) if args.config == "c5" else run_ours(args)
    if Dist().rank == 0:
        print(json.dumps(result), flush=True)
    try:
        import torch.distributed as dist

        if dist.is_initialized():
            dist.barrier()
            dist.destroy_process_group()
    except Exception:  # noqa: BLE001 - teardown only
        pass


if __name__ == "__main__":
    main()
