#!/usr/bin/env python3
"""Benchmark: decoded information Gbps of the framed K=7 rate-1/2 (171,133)
soft-decision Viterbi decoder (BASELINE.json configs[1]: 2^20 overlapping
frames, frame 256, traceback/overlap 42, one B200 per rank).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = decode the rank's whole 2^28-stage int8 LLR stream (2^20 windows
of <=340 stages).  Multi-GPU: one process per GPU (torchrun), each rank owns
its own stream (frames shard with no exchange; weak scaling), timed with CUDA
events, max over ranks.  `value` is device-resident throughput; `e2e` runs the
same decode through the C-ABI host entry (vt_decode_stream_host) with pinned
host buffers, H2D of the LLRs and D2H of the packed bits inside the timed
region.  The reference arm (--impl reference) times the CPU oracle port of the
reference decoder (oracle/, the reference itself is Python and is not
installed on the GPU box) on rank 0 with every host core.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decoded info Gbps per B200 and at 2/4/8 GPUs, K=7 r1/2 soft; BER parity"
K_CODE, GENS, F, V = 7, (0o171, 0o133), 256, 42
N_STAGES = 1 << 28  # 2^20 frames of 256 payload stages
EBN0_DB, SCALE = 3.0, 16.0
PAPER_V100_GBPS = 19.5  # BASELINE.md §1, PAPER.md:797 (V100, fp32 acc / fp32 channel)


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def mark_start(self):
        self.i0 = len(self.lines)

    def mark_end(self):
        time.sleep(0.15)  # the sample taken across the region's end
        self.i1 = len(self.lines)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        # the samples around the timed region: from the last one before it (a short region may
        # hold none of the 100 ms samples) to the first one after it
        i0 = max(0, getattr(self, "i0", 1) - 1)
        i1 = getattr(self, "i1", len(self.lines))
        for ln in self.lines[i0:i1]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def make_stream(torch, n: int, seed: int, device, gens=GENS, k=K_CODE):
    """Synthetic AWGN/BPSK stream generated on the device (SURVEY.md §8(d)
    recipe): random bits -> (171,133) encoder -> BPSK + N(0, sigma^2) at
    Eb/N0 = 3 dB -> q = clamp(rint(16 y), -127, 127) int8, stage-major (N, 2)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    bits = torch.randint(0, 2, (n,), generator=g, device=device, dtype=torch.uint8)
    hist = torch.zeros(n + k - 1, dtype=torch.uint8, device=device)
    hist[k - 1:] = bits
    coded = torch.empty((n, len(gens)), dtype=torch.uint8, device=device)
    for b, gp in enumerate(gens):
        acc = torch.zeros(n, dtype=torch.uint8, device=device)
        for d in range(k):
            if (gp >> (k - 1 - d)) & 1:
                acc ^= hist[k - 1 - d: k - 1 - d + n]
        coded[:, b] = acc
    del hist
    sigma = math.sqrt(1.0 / (2.0 * (1.0 / len(gens)) * 10.0 ** (EBN0_DB / 10.0)))
    q = torch.empty((n, len(gens)), dtype=torch.int8, device=device)
    step = 1 << 24
    for i in range(0, n, step):
        y = 1.0 - 2.0 * coded[i:i + step].float()
        y += sigma * torch.randn(y.shape, generator=g, device=device)
        q[i:i + step] = torch.clamp(torch.round(SCALE * y), -127, 127).to(torch.int8)
    return bits, q


def algorithmic_state_updates(n: int, f: int, v: int, states: int) -> int:
    """Sum over windows of (window length x 2^(K-1)) ACS state updates."""
    nw = -(-n // f)

    def length(w: int) -> int:
        e0 = w * f
        return min(n, min(e0 + f, n) + v) - max(0, e0 - v)

    edges = sorted({w for w in (0, 1, nw - 2, nw - 1) if 0 <= w < nw})
    interior = nw - len(edges)  # all other windows have length f + 2v
    return (sum(length(w) for w in edges) + interior * (f + 2 * v)) * states


def load_peaks() -> dict:
    peaks = {}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peaks.update(json.load(open(p)))
    acs = os.path.join(ROOT, "profiles", "acs_peak.json")
    if os.path.exists(acs):
        peaks["acs"] = json.load(open(acs))
    ncu = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(ncu):
        peaks["ncu"] = json.load(open(ncu))
    return peaks


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_2011_13579_b200 as vt

    ws, rank, local = _dist()
    # VT_BENCH_ONE_GPU=1: every rank on cuda:0 with a gloo process group -- exercises the
    # N>1 flow (barriers, max-over-ranks, rank-0 reporting) on a 1-GPU box; not a bench number
    one_gpu = os.environ.get("VT_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    spec = vt.CodeSpec(K_CODE, GENS)
    n = N_STAGES
    bits_true, q = make_stream(torch, n, seed=1234 + rank, device=dev)
    nwords = (n + 31) // 32
    out = torch.zeros(nwords, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        vt.decode_stream_device(q, spec, F, V, out=out, stream=stream)

    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # the clock sampler starts first (it waits 0.3 s for nvidia-smi): the warm-up steps then
    # run right before the timed ones, so the timed region does not start from idle clocks
    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk.mark_start()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        clk.mark_end()
    if ws > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    red_dev = "cpu" if one_gpu else dev  # (gloo reduces host tensors)
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / args.steps
    value = ws * n / (ms_per_step * 1e-3) / 1e9

    # BER of the decoded stream (sanity) + end-to-end through the C-ABI host entry
    decoded = out.clone()
    ber_err = int(((torch.from_numpy(
        __import__("numpy").unpackbits(decoded.cpu().numpy().view("uint8"), count=n, bitorder="little"))
        .to(dev)) != bits_true).sum().item())
    q_host = q.cpu().pin_memory()
    bits_host = torch.empty(nwords, dtype=torch.int32).pin_memory()
    for _ in range(max(1, min(args.warmup, 2))):
        vt.decode_stream_host(q_host, spec, F, V, bits_host=bits_host, nchunks=args.e2e_chunks, stream=stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e2e_steps = max(1, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        vt.decode_stream_host(q_host, spec, F, V, bits_host=bits_host, nchunks=args.e2e_chunks, stream=stream)
    t_e2e = (time.perf_counter() - t0) / e2e_steps
    te = torch.tensor([t_e2e], dtype=torch.float64, device=red_dev)
    if ws > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = ws * n / float(te.item()) / 1e9
    host_match = bool(torch.equal(bits_host, decoded.cpu()))

    if rank == 0:
        peaks = load_peaks()
        clocks = clk.summary()
        sm_mhz = clocks.get("sm_mhz") or 1900.0
        su = algorithmic_state_updates(n, F, V, 1 << (K_CODE - 1))
        achieved = su / (ms_per_step * 1e-3) / 1e9  # G state-updates/s (one launch per step)
        acs = peaks.get("acs", {})
        per_cyc = acs.get("state_updates_per_cycle_per_sm", {})
        peak_u16 = per_cyc.get("u16x2_viadd_viaddmnmx")
        peak_s32 = per_cyc.get("s32_imad_viaddmnmx")
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        roof = {"bound": "alu", "unit": "Gstate-updates/s", "achieved": round(achieved, 1),
                "traffic": None}
        if peak_u16:
            peak = peak_u16 * sms * sm_mhz * 1e6 / 1e9
            roof.update({"peak": round(peak, 1), "frac": round(achieved / peak, 4),
                         "peak_basis": f"measured ACS microbenchmark (VIADD.16x2+VIADDMNMX.U16x2), "
                                       f"{peak_u16:.1f} state-updates/cycle/SM x {sms} SMs x {sm_mhz:.0f} MHz"})
            if peak_s32:
                roof["frac_vs_s32_form"] = round(achieved / (peak_s32 * sms * sm_mhz * 1e-3), 4)
            loop = acs.get("trellis_loop_su_per_cycle_per_sm", {})
            if loop.get("u16x2_imad_viaddmnmx_acs_bm_groupend_L3"):
                # the same instruction form as the kernel inside a bare trellis loop (no framing,
                # traceback or LLR realignment): the ceiling of this kernel design
                lp = loop["u16x2_imad_viaddmnmx_acs_bm_groupend_L3"] * sms * sm_mhz * 1e-3
                roof["frac_vs_design_loop"] = round(achieved / lp, 4)
        hbm_bytes = n * len(GENS) * (F + 2 * V) / F + n / 8
        hbm_gbs = hbm_bytes / (ms_per_step * 1e-3) / 1e9
        peak_hbm = peaks.get("hbm_gbs", 6554.2)
        roof["secondary"] = {"bound": "hbm", "unit": "GB/s", "achieved": round(hbm_gbs, 1), "peak": peak_hbm,
                             "frac": round(hbm_gbs / peak_hbm, 4),
                             "algorithmic_bytes": "B*(F+2V)/F LLR bytes + 1/8 output byte per info bit"}
        ncu = peaks.get("ncu", {})
        if ncu.get("dram_bytes_per_launch"):
            roof["traffic"] = ncu["dram_bytes_per_launch"]
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "Gbps", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": round(value / PAPER_V100_GBPS, 2),
            "vs_baseline_ref": "paper Table 1: 19.5 Gb/s on V100 (PAPER.md:797), per GPU",
            "dtype": "int8 LLR / packed u16x2 path metrics (K=7 r1/2)", "data": "synthetic AWGN/BPSK, Eb/N0 3 dB, q=clamp(rint(16y))",
            "config": {"workload": "K=7 r1/2 (171,133) soft, 2^20 overlapping frames (F=256, V=42) per GPU, "
                                   "2^28 stages int8 (512 MiB) device-resident; inputs > L2, no flush needed",
                       "code": "K=7 (171,133)", "frame_len": F, "overlap": V, "frames_per_gpu": 1 << 20,
                       "stages_per_gpu": n, "parallelism": f"frames sharded over {ws} GPU(s), no collective"},
            "e2e": {"value": round(e2e_value, 2), "unit": "Gbps", "h2d_bytes_per_step": n * len(GENS),
                    "d2h_bytes_per_step": nwords * 4, "path": "vt_decode_stream_host (C ABI), pinned host buffers",
                    "chunks": args.e2e_chunks, "bits_match_device_path": host_match},
            "roofline": roof,
            "gpu_launches": args.steps,
            "clocks": clocks,
            "ber": {"errors": ber_err, "bits": n, "ber": ber_err / n},
        }
        if not args.no_other_configs and ws == 1:  # (N > 1: the headline only, symmetric teardown)
            line["other_configs"] = other_configs(torch, vt, dev, steps=20)
        if not args.no_cpu_baseline and ws == 1:
            line["cpu_baseline"] = cpu_baseline_full(q_host, decoded, n)
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def other_configs(torch, vt, dev, steps: int) -> list:
    """BASELINE.json configs 3-5 on one GPU (reported beside the headline; not the headline metric)."""
    out = []
    # configs 3 and 4 at the headline's batch (2^20 windows of F=256)
    cases = [("K=7 r1/3 (133,171,165)", 7, (0o133, 0o171, 0o165), 1 << 28, 256, 42),
             ("K=9 r1/2 (753,561)", 9, (0o753, 0o561), 1 << 28, 256, 42),
             ("K=9 r1/2 (753,561) V=54", 9, (0o753, 0o561), 1 << 28, 256, 54)]
    # the headline workload through the other kernel forms (VT_KERNEL_VARIANT)
    cases.append(("K=7 r1/2 F=256 tensor-core branch metrics (16x2tc)", 7, GENS, 1 << 28, 256, 42, "16x2tc"))
    cases.append(("K=7 r1/2 F=256 mma.sync branch metrics (16x2mma)", 7, GENS, 1 << 28, 256, 42, "16x2mma"))
    cases.append(("K=7 r1/2 F=256 one window per thread (s32)", 7, GENS, 1 << 28, 256, 42, "s32"))
    for lw in (16, 18, 22):  # batch sweep at F=256 (2^20 windows is the headline)
        cases.append((f"K=7 r1/2 sweep windows=2^{lw} (F=256)", 7, GENS, 256 << lw, 256, 42))
    for f in (64, 128, 256, 512, 1024):  # frame-length sweep at the headline batch (2^20 windows)
        cases.append((f"K=7 r1/2 sweep F={f} (2^20 windows)", 7, GENS, f << 20, f, 42))
    stream = torch.cuda.current_stream()
    for case in cases:
        label, k, gens, n, f, v = case[:6]
        variant = case[6] if len(case) > 6 else None
        old_env = os.environ.get("VT_KERNEL_VARIANT")
        if variant:
            os.environ["VT_KERNEL_VARIANT"] = variant
        spec = vt.CodeSpec(k, gens)
        bits_true, q = make_stream(torch, n, seed=77, device=dev, gens=gens, k=k)
        o = torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev)
        for _ in range(3):
            vt.decode_stream_device(q, spec, f, v, out=o, stream=stream)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(steps):
            vt.decode_stream_device(q, spec, f, v, out=o, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        su = algorithmic_state_updates(n, f, v, 1 << (k - 1))
        # decoded-bit sanity at Eb/N0 = 3 dB (a kernel regression shows up as a BER jump)
        shifts = torch.arange(32, device=dev, dtype=torch.int32)
        dec = ((o.view(-1, 1) >> shifts) & 1).view(-1)[:n].to(torch.uint8)
        ber = float((dec != bits_true).sum().item()) / n
        out.append({"config": label, "frame_len": f, "overlap": v, "stages": n, "windows": -(-n // f),
                    "value": round(n / (ms * 1e-3) / 1e9, 2), "unit": "Gbps", "ms_per_step": round(ms, 4),
                    "gstate_updates_per_s": round(su / (ms * 1e-3) / 1e9, 1), "ber_3db": ber})
        del dec, bits_true
        if variant:
            if old_env is None:
                os.environ.pop("VT_KERNEL_VARIANT", None)
            else:
                os.environ["VT_KERNEL_VARIANT"] = old_env
        del q, o
    return out


def cpu_baseline_full(q_host, decoded_dev_words, n: int) -> dict:
    """Oracle port of the reference decoder on the host cores, decoding the
    SAME 2^28-stage stream the GPU decoded (all 2^20 windows, ~5 s on 16
    cores); its output is also compared bit-for-bit with the GPU output."""
    import numpy as np

    import oracle

    cores = os.cpu_count() or 1
    qn = q_host.numpy()
    t0 = time.perf_counter()
    ref = oracle.decode_stream(qn, K_CODE, GENS, F, V, threads=cores)
    dt = time.perf_counter() - t0
    gpu = np.unpackbits(decoded_dev_words.cpu().numpy().view(np.uint8), count=n, bitorder="little")
    mism = int(np.count_nonzero(ref != gpu))
    cpu = ""
    try:
        cpu = [ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name")][0]
    except Exception:
        pass
    return {"value": round(n / dt / 1e9, 5), "unit": "Gbps", "cores": cores, "kind": "port",
            "sample": f"the full benchmark stream (2^20 windows, 2^28 info bits) decoded by oracle/viterbi_oracle.c "
                      f"(restatement of reference.decode_batch + framing.decode_stream) in {dt:.1f}s on "
                      f"{cores} threads of {cpu}",
            "parity_vs_gpu": {"bits_compared": n, "mismatches": mism}}


def run_reference(args) -> None:
    """Reference arm: the reference decoder's CPU path (oracle port) on the host."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import numpy as np

    import oracle

    cores = os.cpu_count() or 1
    nwin = 1 << 14
    n = nwin * F + V
    bits, q = oracle.synthetic_stream(n, K_CODE, GENS, ebn0_db=EBN0_DB, seed=1234, scale=SCALE)
    for _ in range(args.warmup):
        oracle.decode_stream(q, K_CODE, GENS, F, V, threads=cores, windows=(0, nwin))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out = oracle.decode_stream(q, K_CODE, GENS, F, V, threads=cores, windows=(0, nwin))
    dt = (time.perf_counter() - t0) / args.steps
    value = nwin * F / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "Gbps", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64 metrics (exact)",
        "data": "synthetic AWGN/BPSK, Eb/N0 3 dB, q=clamp(rint(16y))",
        "config": {"workload": "K=7 r1/2 (171,133) soft, frames F=256 V=42; each step decodes 2^14 frames "
                               "(bounded sample of the 2^20-frame workload)", "frame_len": F, "overlap": V},
        "cpu_baseline": {"value": round(value, 5), "unit": "Gbps", "cores": cores, "kind": "port",
                         "sample": "2^14 windows per step, oracle/viterbi_oracle.c with all host threads"},
        "e2e": {"value": round(value, 5), "unit": "Gbps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "ber": {"errors": int(np.count_nonzero(out[:nwin * F] != bits[:nwin * F])), "bits": nwin * F},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--e2e-chunks", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the extra BASELINE configs (r1/3, K=9, frame-length sweep) reported beside the headline")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
