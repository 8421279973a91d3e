#!/usr/bin/env python3
"""FC-F-OFDM TX+RX throughput on B200 (BASELINE.json metric).

One step = TX synthesis of every local unit (antenna stream x frame) from its
device-resident packed QAM grid, followed by fused RX analysis of every local
unit from the TX waveform.  value = air-interface samples sum_n (N + N_CP,n)
of all units on all ranks / max-over-ranks device time.

  python bench.py [--config c5] [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU: launched by torchrun, one rank per GPU; units are sharded by
(stream, frame) with no data-path collective; the only
collectives are the barrier around the timed region and the max-reduce of the
elapsed time after it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "FC-F-OFDM TX+RX Msamples/s per GPU and at 8 GPUs; % of HBM roofline"
UNIT = "Msamples/s"
SEED = 20080672
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--rx", default="fused", choices=["fused", "direct"])
    ap.add_argument("--units", type=int, default=0, help="override total units (default: the config's)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--dry-run", action="store_true",
                    help="control path only (no GPU): launch/rendezvous, sharding and the final gather on gloo")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def self_launch_cmd(argv: list[str], n: int, port: int) -> list[str]:
    """`bench.py --gpus N` (N > 1) outside torchrun relaunches itself under
    torch.distributed.run, one rank per GPU (127.0.0.1 rendezvous)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def maybe_self_launch(args) -> None:
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket

        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        r = subprocess.run(self_launch_cmd(sys.argv[1:], args.gpus, port))
        sys.exit(r.returncode)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (one rank per GPU)")


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of units for `rank` (first total % world ranks get one more)."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, base + (1 if rank < rem else 0)


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.idx)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ------------------------------------------------------------------ CPU legs
def _banks(w):
    """(Workload, offset) pairs: one for a plain workload, several for a mixed one."""
    return list(zip(w.banks, w.offsets)) if hasattr(w, "banks") else [(w, 0)]


def frame_samples(w) -> int:
    return max(sum(b.N + c for c in b.cp) for b, _ in _banks(w))


def cpu_reference(w, units: int, threads: int, fused: bool, steps: int = 1):
    """The reference's own path (oracle/_ref = unmodified fcwave + FFTW shim) on
    `threads` host threads over `units` whole units.  A mixed workload runs
    each numerology's bank through the reference separately (the reference
    cannot express the mix; the offset sum is negligible).  Returns
    (Msamples/s per step list, kind, sample description)."""
    import oracle as O

    vals = []
    kind = "reference" if O.ref_available() else "port"
    packs = [O.gen_grid(SEED + i, 0, units, b.B, sum(len(x) for x in b.active_maps),
                        w.bits_per_symbol).astype(np.complex64) for i, (b, _) in enumerate(_banks(w))]
    for _ in range(steps):
        t = 0.0
        for (b, _), packed in zip(_banks(w), packs):
            if kind == "reference":
                dt, _chk = O.Ref.bench_txrx(b.N, b.cp, [s.L for s in b.subbands], [s.c for s in b.subbands],
                                            [s.window for s in b.subbands], [len(x) for x in b.active_maps],
                                            b.active_maps, packed, units, threads, simplified=fused)
            else:
                from concurrent.futures import ThreadPoolExecutor

                sys.path.insert(0, os.path.join(ROOT, "tests"))
                from helpers import oracle_rx, oracle_tx

                def one(u, b=b, packed=packed):
                    wv, u0 = oracle_tx(b, packed[u].astype(np.complex128))
                    oracle_rx(b, wv, u0, fused)

                t0 = time.perf_counter()
                with ThreadPoolExecutor(threads) as ex:
                    list(ex.map(one, range(units)))
                dt = time.perf_counter() - t0
            t += dt
        vals.append(units * frame_samples(w) / t / 1e6)
    sample = (f"{units} whole {w.name} units ({', '.join(f'B={b.B}, {len(b.subbands)} subbands' for b, _ in _banks(w))}"
              f"): tx_discontinuous over all subbands + rx_discontinuous per subband "
              f"({'fused' if fused else 'direct'}), one unit per thread; FFT via builder-written FFTW-API shim "
              f"(FFTW3 absent; an FFTW-backed reference would be faster)")
    return vals, kind, sample


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def product_library_loaded() -> bool:
    """Whether this process has the product's CUDA library mapped."""
    try:
        with open("/proc/self/maps") as f:
            return "libfcwave_b200" in f.read()
    except Exception:
        return False


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference_arm(args, w):
    """The reference's own CPU implementation of the path (oracle/_ref: the
    unmodified fcwave sources + FFTW shim) on every host thread, on this arm's
    workload geometry built from the oracle (no product code in this process)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = cpu_threads()
    units = max(1, min(threads, w.units))
    if w.name.startswith("c1"):
        units = max(units, 256)
    vals, kind, sample = cpu_reference(w, units, threads, args.rx == "fused", steps=args.warmup + args.steps)
    timed = vals[args.warmup:] if len(vals) > args.warmup else vals
    value = statistics.mean(timed)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "units": w.units, "units_sampled": units,
                   "sample_note": (f"each step times {units} of the workload's {w.units} units (one whole unit per "
                                   "host thread); the metric is a rate, so the sample measures the same "
                                   "Msamples/s the full workload would run at"),
                   "rx_path": args.rx, "description": w.description},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "cpu_model": cpu_model(), "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_library_loaded": product_library_loaded(),
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
class Runner:
    """Device-resident TX+RX over S local units of a (plain or mixed) workload."""

    def __init__(self, w, S: int, u0: int, dev, fused: bool):
        import torch

        self.w, self.S, self.fused = w, S, fused
        self.mixed = hasattr(w, "banks")
        self.plans = w.plans() if self.mixed else [w.plan()]
        self.mx = w.mixed(self.plans) if self.mixed else None
        self.Q = self.mx.Q if self.mixed else self.plans[0].Q
        banks = w.banks if self.mixed else [w]
        self.grids = []
        for i, (b, p) in enumerate(zip(banks, self.plans)):
            g = torch.empty((S, b.B, p.row_active), dtype=torch.complex64, device=dev)
            p.gen_qam(SEED + i, u0, S, w.bits_per_symbol, g)
            self.grids.append(g)
        self.wave = torch.empty((S, self.Q), dtype=torch.complex64, device=dev)
        self.outs = [torch.empty_like(g) for g in self.grids]
        self.banks = banks

    def tx(self, stream):
        if self.mixed:
            self.mx.tx(self.grids, self.wave, self.S, stream=stream)
        else:
            self.plans[0].tx(self.grids[0], self.wave, self.S, stream=stream)

    def rx(self, stream):
        if self.mixed:
            self.mx.rx(self.wave, self.outs, self.S, fused=self.fused, stream=stream)
        else:
            p = self.plans[0]
            p.rx(self.wave, p.Q, p.useful0, self.outs[0], self.S, fused=self.fused, stream=stream)

    def algorithmic_bytes_per_unit(self) -> dict:
        grid = sum(8 * b.B * p.row_active for b, p in zip(self.banks, self.plans))
        wave = 8 * self.Q
        return {"tx": grid + wave, "rx": grid + wave, "total": 2 * (grid + wave)}

    def e2e(self, n_steps: int, dist, dev, duplex: bool = False) -> float:
        """Seconds per step through the host-buffer public API: grids H2D, TX,
        waveform D2H; waveform H2D, RX, grids D2H (pinned host memory).
        duplex: TX and RX run concurrently on different data (see below)."""
        import torch

        from paper_2008_00672_b200 import PinnedBuffer

        if self.mixed:
            # no host-buffer entry point composes banks: pinned torch copies around the device API
            hg = [g.cpu().pin_memory() for g in self.grids]
            hw = torch.empty(self.wave.shape, dtype=self.wave.dtype).pin_memory()
            ho = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in self.outs]

            def one():
                for d, h in zip(self.grids, hg):
                    d.copy_(h, non_blocking=True)
                self.tx(None)
                hw.copy_(self.wave, non_blocking=True)
                self.wave.copy_(hw, non_blocking=True)
                self.rx(None)
                for h, d in zip(ho, self.outs):
                    h.copy_(d, non_blocking=True)
                torch.cuda.synchronize()
        else:
            p = self.plans[0]
            hg = PinnedBuffer((self.S, self.banks[0].B, p.row_active))
            hw = [PinnedBuffer((self.S, p.Q)), PinnedBuffer((self.S, p.Q))]
            ho = PinnedBuffer((self.S, self.banks[0].B, p.row_active))
            if self.grids is not None:
                self.host_grid = self.grids[0].cpu().numpy()
            hg.array[...] = self.host_grid
            self.grids = self.outs = None
            self.wave = None
            torch.cuda.empty_cache()
            if duplex:
                # full-duplex transceiver: TX of step k (host thread, plan p)
                # overlaps RX of step k-1's waveform (this thread, plan prx);
                # each plan owns its streams and staging, so the two calls
                # load opposite PCIe directions at the same time.
                from concurrent.futures import ThreadPoolExecutor

                prx = self.w.plan()
                pool = ThreadPoolExecutor(1)
                k = [0]
                p.tx_host(hg.array, self.S, out=hw[1].array)

                def one():
                    i = k[0]
                    k[0] += 1
                    fut = pool.submit(p.tx_host, hg.array, self.S, out=hw[i % 2].array)
                    prx.rx_host(hw[(i + 1) % 2].array, p.Q, p.useful0, self.S, fused=self.fused, out=ho.array)
                    fut.result()
            else:
                def one():
                    p.tx_host(hg.array, self.S, out=hw[0].array)
                    p.rx_host(hw[0].array, p.Q, p.useful0, self.S, fused=self.fused, out=ho.array)
        one()  # warm: staging buffers, streams
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(n_steps):
            one()
        return (time.perf_counter() - t0) / n_steps


def flops_per_unit(banks) -> dict:
    """Nominal transform arithmetic of the algorithm as built, 5 n log2 n per
    complex n-point transform (the usual FFT flop convention): per symbol TX
    runs, per subband, the OFDM IDFT_L and the two block DFT_L (ofdm.cpp:97,
    fc_core.cpp:76-90) and, once for all subbands, the two block IFFT_N; fused
    RX runs the two block FFT_N once and, per subband, the IDFT_L / DFT_L pair
    of Eq. (30) (fc_sync.cpp:195-243; direct RX: three L-transforms)."""
    import math

    def t(n):
        return 5.0 * n * math.log2(n)

    tx = rx_f = rx_d = 0.0
    for b in banks:
        sub = sum(t(s.L) for s in b.subbands)
        tx += b.B * (3 * sub + 2 * t(b.N))
        rx_f += b.B * (2 * sub + 2 * t(b.N))
        rx_d += b.B * (3 * sub + 2 * t(b.N))
    return {"tx": tx, "rx_fused": rx_f, "rx_direct": rx_d}


def fp32_peak():
    """Measured FP32 ceiling of this GPU type (tools/ubench_fp32.cu on the box,
    committed as profiles/fp32_peak.json), else the nominal 148 SM x 128 lanes
    x 2 flop x 1.965 GHz."""
    p = os.path.join(ROOT, "profiles", "fp32_peak.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["ffma_tflops"]), "measured (profiles/fp32_peak.json, tools/ubench_fp32.cu FFMA)"
    except Exception:
        return 148 * 128 * 2 * 1.965e9 / 1e12, "nominal (148 SM x 128 FP32 lanes x 2 x 1.965 GHz)"


def knobs() -> dict:
    """FCW_* environment knobs in effect (none are set in a default run)."""
    return {k: v for k, v in os.environ.items() if k.startswith("FCW_")}


def dry_run(args, w) -> None:
    """Control path without a GPU: rendezvous (gloo), sharding, the timing
    max-reduce and the final gather, exactly as the GPU arm runs them."""
    import torch
    import torch.distributed as dist

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    u0, S = shard(w.units, rank, world)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    g = gather_stats(dist if world > 1 else None, torch.tensor([float(u0), float(S), 0.0, 0.0, 0.0, 0.0],
                                                            dtype=torch.float64), world)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "units": w.units, "max_t": float(t.item()),
                          "shards": [[int(r[0]), int(r[1])] for r in g]}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def gather_stats(dist, row, world):
    """Final gather (outside the timed region): every rank's per-shard row."""
    import torch

    if dist is None:
        return [row.tolist()]
    rows = [torch.zeros_like(row) for _ in range(world)]
    dist.all_gather(rows, row)
    return [r.tolist() for r in rows]


def main():
    args = parse()
    maybe_self_launch(args)
    from paper_2008_00672_b200 import configs

    if args.impl == "reference":
        import oracle as O

        # the reference arm builds its geometry from the oracle: no product code loads here
        w = configs.get(args.config, geom=O.Geometry())
        if args.units:
            w.units = args.units
        run_reference_arm(args, w)
        return
    if args.dry_run:
        w = configs.get(args.config, geom=__import__("oracle").Geometry())
        if args.units:
            w.units = args.units
        dry_run(args, w)
        return
    w = configs.get(args.config)
    if args.units:
        w.units = args.units

    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    u0, S = shard(w.units, rank, world)
    dev = torch.device("cuda", local)
    fused = args.rx == "fused"
    run = Runner(w, S, u0, dev, fused)
    stream = torch.cuda.current_stream()

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        run.tx(stream)
        if ev:
            ev[1].record(stream)
        run.rx(stream)
        if ev:
            ev[2].record(stream)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    clk = ClockSampler(local) if rank == 0 else None
    if clk:
        clk.start()
        time.sleep(0.15)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t_end.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = clk.stop() if clk else None
    elapsed_ms = t_start.elapsed_time(t_end)
    tx_ms = [e[0].elapsed_time(e[1]) for e in evs]
    rx_ms = [e[1].elapsed_time(e[2]) for e in evs]
    stats = torch.tensor([elapsed_ms, statistics.mean(tx_ms), statistics.mean(rx_ms)], dtype=torch.float64,
                         device=dev)
    if dist:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    elapsed_ms, tx_avg, rx_avg = [float(x) for x in stats.tolist()]
    ms_per_step = elapsed_ms / args.steps
    total_samples = w.units * frame_samples(w)
    value = total_samples / (ms_per_step * 1e-3) / 1e6

    # final gather (north_star), outside the timed region: per-shard link
    # statistics of the last step's RX output against the seeded transmit bits
    ls_num = ls_den = 0.0
    ls_err = ls_bits = 0
    for i, (b, p) in enumerate(zip(run.banks, run.plans)):
        st = p.link_stats(run.outs[i], S, SEED + i, u0, w.bits_per_symbol, stream=stream)
        ls_num += float(st.evm_num.sum())
        ls_den += float(st.evm_den.sum())
        ls_err += int(st.bit_errors.sum())
        ls_bits += int(st.n_bits.sum())
    rows = gather_stats(dist, torch.tensor([float(u0), float(S), ls_num, ls_den, float(ls_err), float(ls_bits)],
                                           dtype=torch.float64, device=dev), world)

    # roofline of the dominant kernel (algorithmic bytes per launch / mean launch time)
    ab = run.algorithmic_bytes_per_unit()
    peak, peak_src = hbm_peak()
    dom = "rx" if rx_avg > tx_avg else "tx"
    dom_ms = max(rx_avg, tx_avg)
    achieved = ab[dom] * S / (dom_ms * 1e-3) / 1e9
    fl = flops_per_unit(run.banks)
    dom_fl = fl["tx"] if dom == "tx" else fl["rx_fused" if fused else "rx_direct"]
    f_ach = dom_fl * S / (dom_ms * 1e-3) / 1e12
    f_peak, f_src = fp32_peak()
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                t_ent = json.load(f).get(w.name, {}).get(dom)
            if t_ent:
                traffic = t_ent.get("dram_bytes_per_unit", 0) * S
        except Exception:
            traffic = None
    both_gbs = ab["total"] * S / (ms_per_step * 1e-3) / 1e9
    launches_per_step = 2 * len(run.plans)

    e2e = None
    if not args.no_e2e:
        def e2e_time(duplex):
            e = run.e2e(max(1, args.e2e_steps), dist, dev, duplex=duplex)
            t = torch.tensor([e], dtype=torch.float64, device=dev)
            if dist:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())

        serial_s = e2e_time(False)
        duplex_s = e2e_time(True) if not run.mixed else None
        e2e_s = duplex_s if duplex_s is not None else serial_s
        grid_b = (ab["tx"] - 8 * run.Q) * w.units
        wave_b = 8 * run.Q * w.units
        e2e = {"value": total_samples / e2e_s / 1e6, "unit": UNIT, "h2d_bytes_per_step": grid_b + wave_b,
               "d2h_bytes_per_step": wave_b + grid_b, "steps": max(1, args.e2e_steps),
               "path": ("fcw_tx_host + fcw_rx_host (pinned host buffers, 2-stream H2D/kernel/D2H pipeline per "
                        "call); duplex: TX of step k on one host thread overlaps RX of step k-1's waveform on "
                        "another (two plans), so both PCIe directions carry traffic; serial_value: TX then RX"
                        if not run.mixed else "pinned H2D + MixedNumerology.tx/rx + D2H"),
               "serial_value": total_samples / serial_s / 1e6,
               "bound": "PCIe: every step moves the grid and the waveform both ways (profiles/r01/pcie_bw.txt)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = cpu_threads()
        units = max(1, min(threads, w.units))
        vals, kind, sample = cpu_reference(w, units, threads, fused, steps=1)
        cpu = {"value": vals[0], "unit": UNIT, "cores": threads, "cpu_model": cpu_model(), "kind": kind,
               "sample": sample}

    if rank == 0:
        from paper_2008_00672_b200.api import evm_db_from_sums

        N = max(b.N for b in run.banks)
        hbm_frac, fp_frac = achieved / peak, f_ach / f_peak
        g_num, g_den = sum(r[2] for r in rows), sum(r[3] for r in rows)
        g_err, g_bits = int(sum(r[4] for r in rows)), int(sum(r[5] for r in rows))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": w.name, "units": w.units, "units_per_gpu": S,
                       "symbols_per_unit": [b.B for b in run.banks], "subbands": [len(b.subbands) for b in run.banks],
                       "N": [b.N for b in run.banks], "rx_path": args.rx,
                       "l2": "inputs larger than L2 (working set %.1f GB)" % (ab["total"] * w.units / 2 / 1e9)
                       if ab["total"] * w.units / 2 > 126e6 else "working set fits L2 (small config)",
                       "description": w.description, "knobs": knobs()},
            "roofline": {"bound": "hbm" if hbm_frac >= fp_frac else "fp32",
                         "kernel": f"{dom}_kernel<{N}>", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": hbm_frac, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_unit": ab[dom],
                         "txrx_achieved_gbs": both_gbs, "txrx_frac": both_gbs / peak,
                         "fp32": {"achieved": f_ach, "peak": f_peak, "unit": "TFLOP/s", "frac": fp_frac,
                                  "peak_source": f_src, "algorithmic_flops_per_unit": dom_fl,
                                  "model": "5 n log2 n per complex transform (bench.flops_per_unit)",
                                  "ncu": "profiles/r02/SUMMARY.md (IPC, FMA-pipe %)"},
                         "note": ("achieved/peak/frac are the HBM roofline north_star names; bound says which "
                                  "of HBM and FP32 the kernel is closer to")},
            "kernels_ms": {"tx": tx_avg, "rx": rx_avg},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gather": {"ranks": world, "units": int(sum(r[1] for r in rows)),
                       "shards": [[int(r[0]), int(r[1])] for r in rows],
                       "evm_db": evm_db_from_sums(g_num, g_den) if g_den > 0 else None,
                       "bit_errors": g_err, "n_bits": g_bits,
                       "what": "last step's RX grids vs the seeded transmit bits (fcw_link_stats), per shard"},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
