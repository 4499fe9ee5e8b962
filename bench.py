#!/usr/bin/env python
"""bench.py — dropless-MoE layer fwd+bwd throughput on B200 (BASELINE.json metric).

One "step" = one full pass of the hot path over one batch: router, top-k,
topology, padded gather, SDD(+gelu), DSD, weighted scatter, then the backward
pass (scatter-bwd, SDD^T(+gelu'), DS^TD, DSD^T, DD^TS, gather-bwd, router-bwd)
— SURVEY.md §8(a) rows a1..a7, b1..b7. N=1 workload: BASELINE configs[1]
(MoE-XS: T=32768, h=512, f=2048, E=64, top_k=1, bf16, gelu). N>1: expert
parallelism, T=32768 tokens per rank, E=64 experts split over ranks (weak
scaling), NCCL all-to-all dispatch/combine.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes
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
import torch  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
METRIC = "dropless MoE layer fwd+bwd tokens/s"


def load_peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        p["source"] = "measured"
        return p
    except Exception:
        return dict(FALLBACK)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.nvml = None

    # NVML polled every ~2 ms from a thread: the timed region of a default run
    # is only tens of ms, shorter than nvidia-smi's start-up and 100 ms period
    _BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def _nvml_poll(self):
        import pynvml
        while not self._stop:
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.nv.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            phys = self.gpu
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            if vis and all(v.strip().isdigit() for v in vis.split(",")):
                phys = int(vis.split(",")[self.gpu])     # NVML counts physical GPUs
            self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.mx = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.nv, self._stop = [], False
            self.nvml = threading.Thread(target=self._nvml_poll, daemon=True)
            self.nvml.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            time.sleep(0.01)
            self._stop = True
            self.nvml.join(timeout=2)
            sm = [v for v, _ in self.nv]
            reasons = sorted(n for n, b in self._BITS.items() if any(r & b for _, r in self.nv))
            load = [v for v in sm if self.mx and v > 0.5 * self.mx] or sm
            return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": self.mx,
                    "reasons": reasons, "samples": len(sm), "source": "nvml, polled every 2 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        load = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- work model
def work_model(T, h, f, E, k, Tp):
    """Algorithmic FLOPs / bytes per unit."""
    R = T * k
    prod_flop = 2 * R * h * f                       # useful, per product
    prod_bytes = 2 * (R * h + R * f + E * h * f)    # minimal bytes, per product
    return {
        "T": T, "h": h, "E": E, "R": R, "nnz": (Tp // 128) * (f // 128),
        "useful_flop_step": 6 * prod_flop + 2 * T * h * E + 4 * T * h * E,
        "executed_flop_step": 6 * 2 * Tp * h * f,
        "prod_flop": prod_flop,
        "prod_bytes": prod_bytes,
        "sddt_bytes": prod_bytes + 2 * R * f,      # + read of the saved pre-activation H
        "sdd_bytes": prod_bytes,                   # one sparse output
        "sdd_design_bytes": prod_bytes + 2 * R * f,  # this design's SDD also writes act'(H) (reading R18)
        "dsd_scatter_bytes": prod_bytes + 2 * T * h + 4 * R,  # + the gate-weighted rows scattered to y
        # DSD^T writing dx rows instead of dX_g, + dlogits rows and Wr for the router term
        "dsdt_dx_bytes": prod_bytes - 2 * R * h + 2 * T * h + 2 * T * E + 2 * h * E + 4 * R,
        "gather_bytes": 2 * (T * h + R * h) + 4 * R,
        "scatter_bytes": 2 * (R * h + T * h) + 8 * R,
        "scatter_bwd_bytes": 2 * (T * h + 2 * R * h) + 4 * R,
        "gather_bwd_bytes": 2 * (R * h + T * h),
    }


# ----------------------------------------------------------------------------- our arm, 1 GPU
class Step:
    """The layer step as the exact C-ABI call sequence of moe_forward +
    moe_backward (layer.cu), prebuilt ctypes arguments, CUDA events between
    calls so every kernel's time is measured live on the launching stream."""

    def __init__(self, A, cfg, tensors, stream):
        from paper_2211_15841_b200._lib import lib
        self.lib = lib
        self.A = A
        self.cfg = cfg
        t = tensors
        P = ctypes.c_void_p
        c = ctypes.byref(cfg)
        sv = t["saved"]
        topo = ctypes.byref(sv.topo.struct)
        s = P(stream.cuda_stream)
        ws = P(t["ws"].data_ptr())
        d = lambda x: P(x.data_ptr()) if x is not None else None  # noqa: E731
        idn = cfg.act == 0
        L = lib
        wsl = t["ws_layout"]
        self.calls = [
            # router + top-k + topology: one launch where possible (layer.cu: moe_router_topology)
            ("router+topology", L.moe_router_topology, (c, d(t["x"]), d(t["wr"]), d(sv.logits), d(sv.expert_idx),
                                                        d(sv.gates), topo, ws, s)),
        ]
        coded = not idn and sv.act_deriv is None  # layer.cu: only the branch-coded A is saved (R24)
        gfused = bool(L.moe_gather_is_fused(c)) and not coded  # layer.cu: the padded gather inside the SDD / DD^TS loads
        if coded:
            sdd_fwd = ("sdd", L.moe_sdd_act_coded, (c, d(sv.x_g), d(t["w1"]), 0, topo, cfg.act, None, d(sv.a), s))
        else:
            sdd_fwd = ("sdd", L.moe_sdd_deriv, (c, d(sv.x_g), d(t["w1"]), 0, topo, cfg.act, None, d(sv.a),
                                                None if idn else d(sv.act_deriv), s))
        unp = bool(cfg.unpadded)                  # layer.cu: no pad rows, partial blocks at the fringe
        if unp:
            self.calls += [("gather", L.moe_sort_rows, (c, d(t["x"]), topo, d(sv.x_g), s)), sdd_fwd]
        elif gfused:
            self.calls += [("sdd+gather", L.moe_sdd_gather, (c, d(t["x"]), d(t["w1"]), topo, cfg.act, d(sv.a),
                                                            None if idn else d(sv.act_deriv), d(sv.x_g), s))]
        else:
            self.calls += [("gather", L.moe_gather, (c, d(t["x"]), topo, d(sv.x_g), s)), sdd_fwd]
        self.calls += [
            ("dsd+scatter", L.moe_dsd_scatter, (c, d(sv.a), d(t["w2"]), topo, d(sv.gates), d(sv.y_g),
                                                 d(t["y"]), s)),
        ]
        fused =cfg.num_experts % 64 == 0 and cfg.num_experts <= 256 and cfg.top_k <= 8
        if fused and unp:
            bwd = [("scatter_bwd", L.moe_unsort_rows_bwd_router, (c, d(t["dy"]), d(sv.y_g), topo, d(sv.gates),
                                                                  d(sv.logits), d(sv.expert_idx), wsl["dy_g"],
                                                                  wsl["dgates"], wsl["dlogits"], s))]
        elif unp:
            bwd = [("scatter_bwd", L.moe_unsort_rows_bwd, (c, d(t["dy"]), d(sv.y_g), topo, d(sv.gates), wsl["dy_g"],
                                                           wsl["dgates"], s))]
        elif fused:   # moe_backward's tensor-core router path (layer.cu)
            bwd = [("scatter_bwd", L.moe_scatter_bwd_router, (c, d(t["dy"]), d(sv.y_g), topo, d(sv.gates), d(sv.logits),
                                                              d(sv.expert_idx), wsl["dy_g"], wsl["dgates"],
                                                              wsl["dlogits"], s))]
        else:
            bwd = [("scatter_bwd", L.moe_scatter_bwd, (c, d(t["dy"]), d(sv.y_g), topo, d(sv.gates), wsl["dy_g"],
                                                       wsl["dgates"], s))]
        bwd += [
            ("sddT", L.moe_sdd_act_coded, (c, wsl["dy_g"], d(t["w2"]), 1, topo, cfg.act, d(sv.a), wsl["dh"], s))
            if coded else
            ("sddT", L.moe_sdd_deriv, (c, wsl["dy_g"], d(t["w2"]), 1, topo, cfg.act,
                                       None if idn else d(sv.act_deriv), wsl["dh"], None, s)),
            ("dsTd", L.moe_dsd, (c, d(sv.a), 1, wsl["dy_g"], 0, topo, d(t["dw2"]), s)),
        ]
        ddts = (("ddTs+gather", L.moe_dds_gather, (c, d(t["x"]), wsl["dh"], topo, d(t["dw1"]), d(sv.x_g), s)) if gfused
                else ("ddTs", L.moe_dds, (c, d(sv.x_g), 1, wsl["dh"], 0, topo, d(t["dw1"]), s)))
        if fused:   # layer.cu order: DD^TS, dWr, then DSD^T fused with the gather backward + router dx
            bwd += [ddts,
                    ("router_dwr", L.moe_router_dwr, (c, d(t["x"]), wsl["dlogits"], d(t["dwr"]), ws, s)),
                    ("dsdT+dx", L.moe_dsd_dx, (c, wsl["dh"], d(t["w1"]), topo, wsl["dlogits"], d(t["wr"]), d(t["dx"]),
                                               wsl["dx_g"], s))]
        else:
            bwd += [("dsdT", L.moe_dsd, (c, wsl["dh"], 0, d(t["w1"]), 1, topo, wsl["dx_g"], s)),
                    ddts,
                    ("gather_bwd", L.moe_sort_rows_bwd if unp else L.moe_gather_bwd, (c, wsl["dx_g"], topo,
                                                                                        d(t["dx"]), s)),
                    ("router_bwd", L.moe_router_bwd, (c, d(t["x"]), d(t["wr"]), d(sv.logits), d(sv.expert_idx),
                                                      wsl["dgates"], d(t["dwr"]), d(t["dx"]), ws, s))]
        self.calls += bwd
        self.names = [n for n, _, _ in self.calls]

    def run(self, events=None):
        for i, (name, fn, args) in enumerate(self.calls):
            if events is not None:
                events[i].record()
            st = fn(*args)
            if st != 0:
                raise RuntimeError(f"{name}: {self.lib.moe_last_error().decode()}")
        if events is not None:
            events[len(self.calls)].record()


def ws_views(A, cfg, ws):
    """Pointers inside the workspace exactly where moe_backward keeps its
    scratch tensors (moe_workspace_offset)."""
    base = ws.data_ptr()
    off = lambda i: ctypes.c_void_p(base + A.lib.moe_workspace_offset(ctypes.byref(cfg), i))  # noqa: E731
    return {"dy_g": off(0), "dh": off(1), "dx_g": off(2), "dgates": off(3), "dlogits": off(4)}


def flush_l2(buf):
    buf.zero_()


def run_ours_single(args, peaks):
    from paper_2211_15841_b200 import api as A
    from synth import inputs as S

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    shp = S.CONFIGS[args.config]
    T, h, f, E, k = shp.tokens, shp.hidden, shp.ffn, shp.experts, shp.top_k
    inp = S.make_inputs(shp, seed=0)
    cap = A.moe_expert_capacity(T, E, args.capacity_factor) if args.capacity_factor > 0 else 0
    cfg = A.make_config(T, h, E, k, f, act=shp.act, capacity=cap,   # capacity 0: dropless (the headline)
                        unpadded=(args.layout == "unpadded" and not cap))
    stream = torch.cuda.current_stream()
    x = inp["x"].to(dev)
    dy = inp["dy"].to(dev)
    wr, w1, w2 = (inp[n].to(dev) for n in ("wr", "w1", "w2"))
    saved = A.Saved.allocate(cfg, dev, save_deriv=args.act_save == "deriv")
    ws = A.workspace(cfg, dev)
    t = {"x": x, "dy": dy, "wr": wr, "w1": w1, "w2": w2, "saved": saved, "ws": ws,
         "y": torch.empty(T, h, dtype=torch.bfloat16, device=dev),
         "dx": torch.empty(T, h, dtype=torch.bfloat16, device=dev),
         "dwr": torch.empty(h, E, dtype=torch.float32, device=dev),
         "dw1": torch.empty(h, E * f, dtype=torch.bfloat16, device=dev),
         "dw2": torch.empty(E * f, h, dtype=torch.bfloat16, device=dev)}
    t["ws_layout"] = ws_views(A, cfg, ws)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    step = Step(A, cfg, t, stream)
    l2 = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    for _ in range(args.warmup):
        flush_l2(l2)
        step.run()
    torch.cuda.synchronize()
    n = len(step.calls)
    # The step is captured once into a CUDA graph (no host sync inside the
    # layer makes it capturable) with external event-record nodes between the
    # C-ABI calls, so each kernel is still timed on the device; replays remove
    # the per-launch host gaps. Falls back to eager launches if capture fails.
    graph, gev, mode = None, None, "eager"
    if not args.no_graph:
        try:
            gev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(n + 1)]
            l0 = A.lib.moe_total_launch_count()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                step.run(gev)
            launches_per_step = A.lib.moe_total_launch_count() - l0
            graph.replay()
            torch.cuda.synchronize()
            gev[0].elapsed_time(gev[n])
            # the headline: the public API (moe_forward + moe_backward, the calls a
            # user makes; moe_backward forks the router dWr onto a side stream)
            from paper_2211_15841_b200._lib import MoeGrads
            wts = A.weights_struct(t["wr"], t["w1"], t["w2"])
            grd = MoeGrads(t["dwr"].data_ptr(), t["dw1"].data_ptr(), t["dw2"].data_ptr())
            P = ctypes.c_void_p

            def api_step():
                st = A.lib.moe_forward(ctypes.byref(cfg), ctypes.byref(wts), P(t["x"].data_ptr()),
                                       P(t["y"].data_ptr()), ctypes.byref(saved.struct), P(ws.data_ptr()),
                                       P(stream.cuda_stream))
                st = st or A.lib.moe_backward(ctypes.byref(cfg), ctypes.byref(wts), ctypes.byref(saved.struct),
                                              P(t["x"].data_ptr()), P(t["dy"].data_ptr()), P(t["dx"].data_ptr()),
                                              ctypes.byref(grd), P(ws.data_ptr()), P(stream.cuda_stream))
                if st:
                    raise RuntimeError(A.lib.moe_last_error().decode())
            api_step()
            torch.cuda.synchronize()
            l1 = A.lib.moe_total_launch_count()
            graph_plain = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph_plain, stream=stream):
                api_step()
            launches_per_step = A.lib.moe_total_launch_count() - l1
            graph_plain.replay()
            torch.cuda.synchronize()
            mode = "cuda_graph"
        except Exception as exc:  # pragma: no cover - depends on the driver
            print(f"[bench] graph capture unavailable ({exc}); timing eager launches", file=sys.stderr)
            graph = None
            torch.cuda.synchronize()
    launches0 = A.lib.moe_total_launch_count()
    clocks = ClockSampler(dev.index)
    clocks.start()
    torch.cuda.synchronize()
    per_call = np.zeros((args.steps, n))
    step_plain = None
    if graph is not None:
        # (1) headline: whole steps, events only around each step
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        for i in range(args.steps):
            flush_l2(l2)                      # between timed steps, outside the events
            ev0[i].record(stream)
            graph_plain.replay()
            ev1[i].record(stream)
        torch.cuda.synchronize()
        step_plain = np.array([ev0[i].elapsed_time(ev1[i]) for i in range(args.steps)])
        # (2) breakdown: the same step with an event node between the C-ABI calls
        for i in range(args.steps):
            flush_l2(l2)
            graph.replay()
            torch.cuda.synchronize()
            per_call[i] = [gev[j].elapsed_time(gev[j + 1]) for j in range(n)]
        launches = launches_per_step * args.steps
    else:
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n + 1)] for _ in range(args.steps)]
        for i in range(args.steps):
            flush_l2(l2)
            step.run(evs[i])
        torch.cuda.synchronize()
        launches = A.lib.moe_total_launch_count() - launches0
        per_call = np.array([[evs[i][j].elapsed_time(evs[i][j + 1]) for j in range(n)] for i in range(args.steps)])
    torch.cuda.synchronize()
    clk = clocks.stop()
    step_ms = step_plain if step_plain is not None else per_call.sum(axis=1)
    total_ms = float(step_ms.sum())
    Tp, nnz = saved.topo.sizes()
    counts = saved.topo["counts"].cpu().numpy()
    value = T * args.steps / (total_ms / 1e3)

    # ---- roofline for the dominant kernel (largest share of the step)
    wm = work_model(T, h, f, E, k, Tp)
    mean_call = per_call.mean(axis=0)
    shares = mean_call / mean_call.sum()
    dom = int(np.argmax(mean_call))
    dname = step.names[dom]
    prod_names = {"sdd": "sdd_bytes", "sdd+gather": "sdd_bytes", "ddTs+gather": "prod_bytes",
                  "dsd+scatter": "dsd_scatter_bytes", "sddT": "sddt_bytes", "dsTd": "prod_bytes",
                  "dsdT": "prod_bytes", "ddTs": "prod_bytes", "dsdT+dx": "dsdt_dx_bytes"}
    byte_names = {"gather": "gather_bytes", "scatter": "scatter_bytes", "scatter_bwd": "scatter_bwd_bytes",
                  "gather_bwd": "gather_bwd_bytes"}
    dur_s = mean_call[dom] / 1e3
    roof = {"kernel": dname, "launch_ms": round(float(mean_call[dom]), 4), "share_of_step": round(float(shares[dom]), 4)}
    kinfo = kernel_roofline(dname, wm, dur_s, peaks, prod_names, byte_names)
    roof.update({kk: vv for kk, vv in kinfo.items() if kk != "ms"})
    roof["peak_source"] = peaks.get("source", "measured") + " (burst)"
    tr = load_traffic(dname)
    roof["traffic"] = tr.get("bytes") if tr else None
    if tr:
        roof["traffic_source"] = tr.get("source")
    coded = cfg.act != 0 and saved.act_deriv is None
    roof["saved_for_backward"] = ("branch-coded A only (R24): the SDD writes one output, the §8(d) bytes" if coded
                                  else "A and act'(H) (R18)")
    if dname == "sdd" and not coded:
        # this design writes act(H) AND act'(H) (reading R18): the same launch
        # against its own two-output byte count, beside the §8(d) figure above
        b2 = wm["sdd_design_bytes"]
        roof["design_two_outputs"] = {"bytes": b2, "achieved": round(b2 / dur_s / 1e9, 1),
                                      "frac": round(b2 / dur_s / 1e9 / peaks["hbm_gbs"], 4)}
    if dname == "sdd":
        # context: bytes the SDD moves through the SMs' TMA ports.
        # The default CTA-pair kernel: per 256 x 256 pair tile each CTA loads
        # its 128 rows of X_g and 128 columns of W1 (2 x 128 x h bf16 each) and
        # stores its 128 x 256 share of act(H) and act'(H); an expert's lone
        # last block-row runs as an M = 128 pair tile (64 rows per CTA, same
        # loads, half the stores). Against the measured TMA L2->SMEM ceiling
        # (scripts/micro/l2_tma_bw.cu, profiles/r1s5_l2_tma_bw.txt).
        brows = (counts + 127) // 128
        full_pairs, half_pairs = int((brows // 2).sum()), int((brows % 2).sum())
        F = f // 128
        outs = 1 if coded else 2
        per_cta_load = 2 * (128 * h + 128 * h)
        per_cta_store = outs * 2 * 128 * 256
        pair_kernel = T * k >= 3 * E * 128 and F % 2 == 0 and h % 256 == 0 and os.environ.get("MOE_SDD_PAIR", "") != "0"
        if pair_kernel:
            port_bytes = (full_pairs + half_pairs) * (F // 2) * 2 * per_cta_load \
                + (full_pairs + 0.5 * half_pairs) * (F // 2) * 2 * per_cta_store
            tiles = {"pair_tiles": (full_pairs + half_pairs) * (F // 2), "half_pair_tiles": half_pairs * (F // 2)}
        else:  # 1-SM 128 x 256 tiles: A (128 x h) and B (h x 256) in, the outputs out
            port_bytes = (nnz // 2) * (2 * (128 * h + h * 256) + outs * 2 * 128 * 256)
            tiles = {"tiles_1sm": nnz // 2}
        feed = port_bytes / dur_s / 1e12
        roof["sm_port"] = {"bytes": int(port_bytes), **tiles, "achieved_tbs": round(feed, 2),
                           "tma_l2_to_smem_ceiling_tbs": 14.59, "frac": round(feed / 14.59, 3)}
    breakdown = {nm: {"ms": round(float(m), 4), "share": round(float(s_), 4),
                      **kernel_roofline(nm, wm, m / 1e3, peaks, prod_names, byte_names)}
                 for nm, m, s_ in zip(step.names, mean_call, shares)}
    gemm_ms = sum(mean_call[step.names.index(p)] for p in prod_names if p in step.names)
    gemm = {"ms": round(float(gemm_ms), 4),
            "useful_tflops": round(6 * wm["prod_flop"] / (gemm_ms / 1e3) / 1e12, 1),
            "executed_tflops": round(wm["executed_flop_step"] / (gemm_ms / 1e3) / 1e12, 1)}
    gemm["frac_of_bf16_peak"] = round(gemm["useful_tflops"] / peaks["bf16_tflops"], 4)

    e2e = run_e2e(A, cfg, t, args, dev) if not args.no_e2e else None
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) inputs, "
        "random-init weights of the MoE-XS shape)",
        "config": {"workload": shp.name, "tokens": T, "hidden": h, "ffn_hidden": f, "num_experts": E, "top_k": k,
                   "block_size": 128, "act": "gelu_tanh", "routing": shp.routing, "parallelism": "ep1",
                   "padded_rows": Tp, "nnz_blocks": nnz,
                   "layout": "unpadded (partial blocks at the fringe, P:297)" if cfg.unpadded else "padded (P:297)",
                   "expert_load_max_over_mean": round(float(counts.max() / counts.mean()), 3),
                   **({"formulation": "token-dropping", "capacity_factor": args.capacity_factor, "capacity": cap,
                       "dropped_fraction": round(1.0 - float(counts.sum()) / (T * k), 4)} if cap else
                      {"formulation": "dropless"}),
                   "l2": "flushed between timed steps (512 MiB memset, outside the events)"},
        "roofline": roof,
        "gemm": gemm,
        "breakdown_ms": breakdown,
        "breakdown_note": "value/ms_per_step: CUDA-graph replays of moe_forward + moe_backward (the public "
                          "API; the router dWr runs on a side stream beside the SDD^T). breakdown_ms: a second "
                          "replay of the same kernels as individual C-ABI calls in layer.cu order, serialised, "
                          "with an event node between calls (sum %.4f ms/step incl. the event gaps)"
                          % float(per_call.sum(axis=1).mean()),
        "clocks": clk,
        "launch_mode": mode,
        "gpu_launches": int(launches),
        "e2e": e2e,
    }
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(shp)
    return out


def kernel_roofline(name, wm, dur_s, peaks, prod_names, byte_names):
    """Roofline entry of one launch: SURVEY §8(d) algorithmic bytes (and FLOPs
    for the products) / its event-timed duration, against the measured peaks.
    The router and topology are reported against HBM too (the topology is
    latency-bound: a tiny frac is expected)."""
    T, h, E, R = wm["T"], wm["h"], wm["E"], wm["R"]
    extra = {"router": 2 * T * h + 4 * T * E + 8 * R + 2 * h * E,
             "router+topology": 2 * T * h + 4 * T * E + 8 * R + 2 * h * E + 12 * R + 12 * wm["nnz"],
             "router_dwr": 2 * T * h + 2 * T * E + 4 * h * E,
             "topology": 12 * R + 12 * wm["nnz"]}
    out = {}
    if dur_s <= 0:
        return out
    if name in prod_names:
        bytes_ = wm[prod_names[name]]
        flop = wm["prod_flop"]
        t_mem, t_flop = bytes_ / (peaks["hbm_gbs"] * 1e9), flop / (peaks["bf16_tflops"] * 1e12)
        if t_mem >= t_flop:
            out.update(bound="hbm", achieved=round(bytes_ / dur_s / 1e9, 1), peak=peaks["hbm_gbs"], unit="GB/s")
        else:
            out.update(bound="tensor", achieved=round(flop / dur_s / 1e12, 1), peak=peaks["bf16_tflops"],
                       unit="TFLOP/s")
        out["alg_bytes"] = int(bytes_)
        out["tflops_useful"] = round(flop / dur_s / 1e12, 1)
        out["tflops_frac_of_bf16_peak"] = round(flop / dur_s / 1e12 / peaks["bf16_tflops"], 4)
    elif name in byte_names or name in extra:
        bytes_ = wm[byte_names[name]] if name in byte_names else extra[name]
        out.update(bound="hbm", achieved=round(bytes_ / dur_s / 1e9, 1), peak=peaks["hbm_gbs"], unit="GB/s",
                   alg_bytes=int(bytes_))
    if out.get("achieved") is not None:
        out["frac"] = round(out["achieved"] / out["peak"], 4)
    return out


def load_traffic(kernel_name):
    """dram bytes per launch for the dominant kernel from the committed ncu
    --set full capture summary (profiles/traffic.json, which names its capture
    and date), else null. ncu cannot run inside the timed bench, so this is the
    latest committed capture of the same kernel, stamped with its source."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        v = d.get(kernel_name)
        if v is None:
            return None
        return {"bytes": v, "source": d.get("source", "profiles/traffic.json")}
    except Exception:
        return None


def run_e2e(A, cfg, t, args, dev):
    """Same metric through the public API (moe_forward + moe_backward) with
    pinned HOST inputs copied in and results (y, dx) copied out every step."""
    T, h = cfg.tokens, cfg.hidden
    hx = t["x"].cpu().pin_memory()
    hdy = t["dy"].cpu().pin_memory()
    hy = [torch.empty(T, h, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    hdx = [torch.empty(T, h, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    xd = [torch.empty_like(t["x"]) for _ in range(2)]
    dyd = [torch.empty_like(t["dy"]) for _ in range(2)]
    yd = [torch.empty_like(t["y"]) for _ in range(2)]
    dxd = [torch.empty_like(t["dx"]) for _ in range(2)]
    saved, ws = t["saved"], t["ws"]
    grads = (t["dwr"], t["dw1"], t["dw2"])
    # three streams: host->device copies of step i+1 and device->host copies
    # of step i-1 overlap step i's compute (double-buffered device tensors)
    s_in, s_c, s_out = torch.cuda.Stream(), torch.cuda.current_stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    for b in range(2):
        ev_comp[b].record(s_c)
        ev_out[b].record(s_out)

    def one(i):
        b = i & 1
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_comp[b])           # step i-2 finished reading xd[b], dyd[b]
            xd[b].copy_(hx, non_blocking=True)
            dyd[b].copy_(hdy, non_blocking=True)
            ev_in[b].record(s_in)
        with torch.cuda.stream(s_c):
            s_c.wait_event(ev_in[b])
            s_c.wait_event(ev_out[b])             # step i-2's results left yd[b], dxd[b]
            y, _ = A.moe_forward(cfg, t["wr"], t["w1"], t["w2"], xd[b], y=yd[b], saved=saved, ws=ws)
            dx, _ = A.moe_backward(cfg, t["wr"], t["w1"], t["w2"], saved, xd[b], dyd[b], dx=dxd[b], grads=grads,
                                   ws=ws)
            ev_comp[b].record(s_c)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_comp[b])
            hy[b].copy_(y, non_blocking=True)
            hdx[b].copy_(dx, non_blocking=True)
            ev_out[b].record(s_out)

    for i in range(max(1, args.warmup)):
        one(i)
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record(s_in)
    for i in range(args.steps):
        one(i)
    s_out.wait_stream(s_c)
    en.record(s_out)
    torch.cuda.synchronize()
    ms = st.elapsed_time(en)
    return {"value": round(T * args.steps / (ms / 1e3), 1), "unit": "tokens/s",
            "h2d_bytes_per_step": 2 * T * h * 2, "d2h_bytes_per_step": 2 * T * h * 2,
            "ms_per_step": round(ms / args.steps, 4),
            "api": "moe_forward+moe_backward (C ABI); pinned host x, dy in and y, dx out every step, copies "
                   "on separate streams overlapping the neighbouring steps' compute"}


# ----------------------------------------------------------------------------- oracle timings
def oracle_step(inp, shp, T_sample):
    from oracle import moe_oracle as O
    from synth import inputs as S
    x, wr, w1, w2, dy = (S.to_f64(inp[n][:T_sample]) if n in ("x", "dy") else S.to_f64(inp[n])
                         for n in ("x", "wr", "w1", "w2", "dy"))
    y, cache = O.dmoe_forward(x, wr, w1, w2, shp.top_k, 128, shp.ffn, shp.act)
    O.dmoe_backward(cache, dy, wr, w1, w2)


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads") for i in threadpool_info() if i.get("internal_api") == "openblas"]
        if n:
            return int(n[0])
    except Exception:
        pass
    return os.cpu_count()


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(shp, T_sample=None):
    """The oracle as it stands, one fwd+bwd of the whole bench workload (all
    T tokens: no extrapolation) on the host cores."""
    from synth import inputs as S
    T_sample = T_sample or shp.tokens
    inp = S.make_inputs(shp, seed=0, tokens=T_sample)
    t0 = time.perf_counter()
    oracle_step(inp, shp, T_sample)
    dt = time.perf_counter() - t0
    return {"value": round(T_sample / dt, 1), "unit": "tokens/s", "cores": cpu_threads(), "kind": "oracle",
            "nproc": os.cpu_count(), "cpu_model": cpu_model(),
            "sample": f"all {T_sample} tokens of the {shp.name} workload, one fwd+bwd of oracle/moe_oracle.py "
                      f"(numpy fp64, OpenBLAS matmul per block) in {dt:.2f} s"}


def run_reference(args):
    from synth import inputs as S
    shp = S.CONFIGS[args.config]
    T_sample = args.ref_tokens
    inp = S.make_inputs(shp, seed=0, tokens=T_sample)
    for _ in range(args.warmup):
        oracle_step(inp, shp, T_sample)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_step(inp, shp, T_sample)
    dt = time.perf_counter() - t0
    value = T_sample * args.steps / dt
    return {"impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": "tokens/s", "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": shp.name, "tokens_per_step_sample": T_sample,
                                           "hidden": shp.hidden, "ffn_hidden": shp.ffn,
                                           "num_experts": shp.experts, "top_k": shp.top_k},
            "cpu_baseline": {"value": round(value, 2), "unit": "tokens/s", "cores": cpu_threads(), "kind": "oracle",
                             "nproc": os.cpu_count(), "cpu_model": cpu_model(),
                             "sample": f"{T_sample} tokens of {shp.name} per step (full h, f, E)"},
            "e2e": {"value": round(value, 2), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-tokens", type=int, default=4096)
    ap.add_argument("--ep", action="store_true", help="expert-parallel path even at one rank")
    ap.add_argument("--capacity-factor", type=float, default=0.0,
                    help="> 0: time the token-dropping formulation (P:112-116) with this capacity factor "
                         "instead of the dropless layer (context only; the headline is dropless)")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a CUDA graph")
    ap.add_argument("--act-save", default=os.environ.get("MOE_BENCH_ACT_SAVE", "deriv"), choices=["coded", "deriv"],
                    help="what the forward saves for the SDD^T: act'(H) beside A (R18, default) or the "
                         "branch-coded A alone (R24: one buffer less, measured slower)")
    ap.add_argument("--layout", default=os.environ.get("MOE_BENCH_LAYOUT", "padded"), choices=["padded", "unpadded"],
                    help="dense expert-grouped rows padded to 128 per expert (P:297, the paper's layout) or not "
                         "(partial blocks at the fringe, NEXT-3); same outputs")
    ap.add_argument("--transport", default=os.environ.get("MOE_EP_TRANSPORT", "auto"), choices=["auto", "nccl", "p2p"],
                    help="expert-parallel token exchange: device-initiated peer stores (p2p; auto = p2p with an "
                         "NCCL fallback if peer memory is unusable) or NCCL all-to-all")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    # NCCL's version / debug lines go to stderr so stdout carries only the JSON line:
    # native libraries print to fd 1 directly (NCCL's "NCCL version" line ignores
    # NCCL_DEBUG_FILE), so fd 1 is pointed at stderr and the JSON goes to a dup
    # of the original stdout.
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    sys.stdout.flush()
    out_fd = os.dup(1)
    os.dup2(2, 1)
    emit = os.fdopen(out_fd, "w")

    def print(line, flush=True):  # noqa: A001 - the one JSON line, to the real stdout
        emit.write(line + "\n")
        emit.flush()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    peaks = load_peaks()
    if world > 1 or args.ep:
        from paper_2211_15841_b200 import ep
        out = ep.bench_ep(args, peaks, ClockSampler)
        if rank == 0 and out is not None:
            print(json.dumps(out), flush=True)
        return
    out = run_ours_single(args, peaks)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
