#!/usr/bin/env python3
"""Benchmark: decode tokens/s of the Llama-2-7B-shaped integer model (BASELINE.json
configs[1]: 7B-shaped random-init int8 weights, seed 7; ChaCha20 prompt seed 8,
16 tokens; batch-1 greedy decode) on N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one greedy decode token: one full forward of the 32-layer model
(6.62 GB of int8 weights + scales) plus the argmax that appends the next token.

  N = 1   the persistent decode kernel (one launch for all K steps).
  N > 1   (torchrun, one process per GPU) TENSOR PARALLEL decode of the same
          single sequence (BASELINE configs[3]): each rank holds
          1/N of every matrix and runs the persistent decode kernel on it;
          the pre-scale WO / w_down accumulators (uint64 sums) and the
          lm_head argmax pairs are exchanged INSIDE that kernel over NVLink
          peer memory (backend "fused-ipc": CUDA IPC handles gathered over
          torch.distributed, no collective call per layer);
          value = K / max-over-ranks time (strong scaling: the work per token
          is fixed, each GPU streams 1/N of it). The tokens are checked
          against the C2 golden. Extra keys at N > 1:
            tp_nccl  the same decode with per-stage GEMVs + NCCL all-reduce
                     (the collective-library baseline)
            c5  every rank generates its 8 C5 sequences through the batch
                call (seqs 8r .. 8r+7), per-sequence hashes vs the goldens
            dp  every rank decodes its own sequence with the single-GPU
                kernel (weak-scaling replicas, the N = 1 kernel's aggregate)
          At N = 1, tp_one_gpu: the fused group program for g = 2, 4, 8 with
          all g shards on this one GPU (one cooperative launch, ranks share
          its HBM and SMs): the in-kernel exchange's cost, not a scaling figure.

Keys beyond the base contract:
  e2e           the same metric through the reference-shaped C-ABI call
                (dimg_generate_greedy / dimg_tp_generate_greedy) with HOST
                buffers: prompt H2D, tokens D2H and the BLAKE3 hash inside
                the timed region
  roofline      the dominant kernel per decode step: algorithmic bytes per
                step (per GPU at N > 1) / CUDA-event step time, vs
                MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the reference engine (oracle/_ref, compiled from its own
                sources) timed on this host, rank 0, N=1
--impl reference times that reference engine alone on the same workload
(same prompt, same decode positions, same config dict).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG7B = (32, 4096, 32, 11008, 32000, 4096)
MODEL_SEED = 7
PROMPT_SEED = 8
PROMPT_LEN = 16
WEIGHT_HASH_7B = "8df01f77395ece3685b121f642da4442bda0862a3e76cc9823577ffc5880dd64"
METRIC = "decode tokens/s (Llama-2-7B int) at 1/2/4/8 B200; 0 hash mismatches vs CPU"


def bytes_per_token(L, D, F, V):
    """Algorithmic HBM bytes of one decode forward: int8
    weights incl. lm_head + int64 row scales + int64 norm gains + one
    embedding row (int8 row + its int64 scale). KV traffic excluded."""
    w = L * (4 * D * D + 3 * D * F) + V * D
    s = L * (4 * D + 2 * F + D) + V
    g = (2 * L + 1) * D
    return w + 8 * s + 8 * g + D + 8


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _pci_bus_id(cuda_index):
    """PCI bus id of CUDA device `cuda_index` (NVML numbers GPUs differently
    when CUDA_VISIBLE_DEVICES is set)."""
    import ctypes
    cu = ctypes.CDLL("libcuda.so.1")
    cu.cuInit(0)
    buf = ctypes.create_string_buffer(64)
    if cu.cuDeviceGetPCIBusId(buf, 64, cuda_index) != 0:
        return None
    return buf.value.decode()


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML
    every ~2 ms from a thread (a 35 ms decode region still gets ~15
    samples); nvidia-smi (~50 ms per call) if NVML is unavailable."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, set of reason names)
        self.source = None
        self._stop = threading.Event()
        self._t = None
        self._nv = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            bus = _pci_bus_id(index)
            h = nv.nvmlDeviceGetHandleByPciBusId(bus) if bus else nv.nvmlDeviceGetHandleByIndex(index)
            self._nv, self._h = nv, h
            self._bits = [(nv.nvmlClocksEventReasonHwSlowdown, "hw_slowdown"),
                          (nv.nvmlClocksEventReasonHwThermalSlowdown, "hw_thermal_slowdown"),
                          (nv.nvmlClocksEventReasonSwThermalSlowdown, "sw_thermal_slowdown"),
                          (nv.nvmlClocksEventReasonSwPowerCap, "sw_power_cap")]
            self._max = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.source = "nvml"
        except Exception:
            self._nv = None
            self.source = "nvidia-smi"

    def _sample_nvml(self):
        nv, h = self._nv, self._h
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        self.rows.append((float(sm), float(self._max), {n for b, n in self._bits if r & b}))

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True,
                             text=True, timeout=5).stdout.strip()
        if out:
            r = [c.strip() for c in out.split(",")]
            if r[1].replace(".", "").isdigit():
                mx = float(r[2]) if r[2].replace(".", "").isdigit() else None
                self.rows.append((float(r[1]), mx, {self.NAMES[i] for i in range(4)
                                                    if len(r) > 5 + i and r[5 + i].lower() == "active"}))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample_nvml() if self._nv else self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.002 if self._nv else 0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        if not self.rows:  # the region was shorter than one sample: take one now
            try:
                self._sample_nvml() if self._nv else self._sample_smi()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(r[0] for r in self.rows)
        mx = max((r[1] for r in self.rows if r[1]), default=None)
        reasons = sorted(set().union(*(r[2] for r in self.rows)))
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows), "sm_mhz_min": sm[0], "source": self.source}


# --------------------------------------------------------------------------
def host_cpu():
    """nproc and the CPU model of this host (SURVEY §8d asks for both)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def config_dict(world, extra=None):
    """The workload description both arms print (same_config)."""
    d = {"workload": "C2: Llama-2-7B-shaped int8/Q16 model, batch-1 greedy decode",
         "model": "llama2-7b-shaped-int", "layers": CFG7B[0], "d_model": CFG7B[1], "d_ffn": CFG7B[3],
         "vocab": CFG7B[4], "seed": MODEL_SEED, "prompt_seed": PROMPT_SEED, "prompt_len": PROMPT_LEN,
         "decode_positions": "15+W .. 14+W+K (after the 15 prompt positions and W warm-up steps)",
         "global_batch": 1, "parallelism": f"tp{world}" if world > 1 else "single GPU",
         "l2": "weights 6.6 GB/step > 126 MB L2 (no flush needed)"}
    d.update(extra or {})
    return d


def reference_model(ref, cfg):
    """The reference's own gen_toy_model (proj/src/model.cpp:189-215)."""
    return ref.gen_toy(MODEL_SEED, cfg)


def time_reference(ref, m, n_warm, n_timed, prompt, threads):
    """Greedy decode through dim::InferenceSession::forward (+select_greedy),
    the reference's stock path: prompt[:-1] untimed, then the decode steps
    (the first one feeds prompt[-1]) -- the GPU arm's positions. Returns
    (seconds per decode forward, tokens of the warm + timed steps)."""
    import ctypes as C
    h = C.c_void_p()
    assert ref.lib.ref_session_new(m.h, threads, C.byref(h)) == 0
    nxt = C.c_uint32()
    pos = 0
    for t in prompt[:-1]:  # prefill (untimed)
        assert ref.lib.ref_session_forward(h, int(t), pos, None, C.byref(nxt)) == 0
        pos += 1
    tok, toks = int(prompt[-1]), []
    for _ in range(n_warm):
        assert ref.lib.ref_session_forward(h, tok, pos, None, C.byref(nxt)) == 0
        tok = nxt.value
        toks.append(tok)
        pos += 1
    t0 = time.perf_counter()
    for _ in range(n_timed):
        assert ref.lib.ref_session_forward(h, tok, pos, None, C.byref(nxt)) == 0
        tok = nxt.value
        toks.append(tok)
        pos += 1
    dt = time.perf_counter() - t0
    ref.lib.ref_session_free(h)
    return dt / max(1, n_timed), toks


def golden_c2():
    try:
        with open(os.path.join(ROOT, "tests", "golden", "models_7b.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from oracle.pyoracle import Config, Reference
    cfg = Config(*CFG7B)
    threads = os.cpu_count() or 1
    if not Reference.available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/libdimref.so not built"})
        return 0
    ref = Reference()
    t0 = time.time()
    m = reference_model(ref, cfg)
    gen_s = time.time() - t0
    prompt = ref.prompt(PROMPT_SEED, cfg.vocab, PROMPT_LEN)
    spf, toks = time_reference(ref, m, args.warmup, args.steps, prompt, threads)
    gold = golden_c2().get("c2", {}).get("tokens", [])
    n = min(len(toks), len(gold))
    value = 1.0 / spf
    sample = (f"dim::InferenceSession::forward + select_greedy: the 16-token prompt's first 15 positions "
              f"untimed, {args.warmup} warm-up and {args.steps} timed decode forwards (threads={threads}; "
              f"the reference's dense matvec is single-threaded, so 1 core does the work)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": spf * 1e3, "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic (reference gen_toy_model seed 7)",
        "config": config_dict(world),
        "tokens_match_c2_golden": toks[:n] == gold[:n] if n else None,
        "cpu_baseline": dict({"value": value, "unit": "tokens/s", "cores": 1, "kind": "reference",
                              "sample": sample, "threads_setting": threads, "model_gen_s": round(gen_s, 1)},
                             **host_cpu()),
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# --------------------------------------------------------------------------
def cpu_baseline(model_file, cfg_t):
    """Reference engine on this host over the SAME weights (bounded sample:
    a 2-token prompt, then 10 timed decode forwards, threads=1)."""
    try:
        from oracle.pyoracle import Config, Reference
        if not Reference.available():
            raise FileNotFoundError("oracle/_ref not built")
        ref = Reference()
        cfg = Config(*cfg_t)
        import numpy as np
        names = ["tok_embd"] + [f"layers.{l}.{t}" for l in range(cfg.n_layers)
                                for t in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")] + ["output"]
        w = np.concatenate([model_file.tensor(n)[0].reshape(-1) for n in names])
        s = np.concatenate([model_file.tensor(n)[1] for n in names])
        m = ref.model_from_arrays(cfg, w, s, model_file.norms())
        del w, s
        prompt = ref.prompt(PROMPT_SEED, cfg.vocab, PROMPT_LEN)[:2]
        spf, _ = time_reference(ref, m, 0, 10, prompt, 1)
        return dict({"value": 1.0 / spf, "unit": "tokens/s", "cores": 1, "kind": "reference",
                     "sample": "10 timed decode forwards (dim::InferenceSession::forward + select_greedy) after "
                               "a 2-token prompt, same weights, threads=1 (the dense matvec is single-threaded)"},
                    **host_cpu())
    except Exception as e:  # reported, never fatal for the GPU number
        return {"value": None, "unit": "tokens/s", "cores": 1, "kind": "reference",
                "sample": f"unavailable: {e}"}


def mma_i8_peak():
    """Measured dense kind::i8 tcgen05 rate (profiles/r02_mma_rate.json,
    tools/mma_rate.cu on this pool's B200), else 2 x the bf16 burst."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_mma_rate.json")) as f:
            d = json.load(f)
        return float(d["i8_tops"]), "measured kind::i8 tcgen05.mma rate (profiles/r02_mma_rate.json)"
    except Exception:
        pass
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return 2 * json.load(f)["bf16_tflops"], "2 x measured bf16 burst (kind::i8 at twice kind::f16)"
    except Exception:
        return 2 * 1590.0, "2 x fallback bf16"


def c3_algorithmic_ops(cfg, T):
    """2 x the int8 MACs of every layer GEMM at T tokens + the
    last position's lm_head + the causal attention's QK^T and PV."""
    L, D, F, V, H = cfg.n_layers, cfg.d_model, cfg.d_ffn, cfg.vocab, cfg.n_heads
    dh = D // H
    return 2 * L * (4 * D * D + 3 * D * F) * T + 2 * V * D + 2 * 2 * L * H * dh * T * (T + 1) // 2


def prefill_c3(P, mf, cfg, dev):
    """C3: prefill of a 2048-token synthetic prompt (prompt seed 9): positions
    0..2046 through every layer on the tensor cores (dimg_session_time_prefill)
    plus the last prompt position's decode step that yields the first token
    (dimg_session_time_decode), both CUDA-event timed; 2 warm + 3 timed,
    median. Roofline: the ALGORITHMIC int8 ops of the whole 2048-token prefill
    (2.763e13) per second against the measured kind::i8 rate."""
    try:
        n_prompt = 2048
        prompt = P.prompt_from_seed(9, cfg.vocab, n_prompt)
        s = P.InferenceSession(mf, P.EngineOptions(device=dev))
        times, tc = [], True
        for i in range(5):
            s.begin(prompt, 1)
            ms, used = s.time_prefill()
            ms += s.time_decode(1)
            tc &= used
            if i >= 2:
                times.append(ms)
        ms = sorted(times)[len(times) // 2]
        ops = c3_algorithmic_ops(cfg, n_prompt)
        peak, kind = mma_i8_peak()
        tops = ops / (ms / 1e3) / 1e12
        first = s.tokens(1)[0]
        gold = golden_c2().get("c3", {}).get("tokens", [None])[0]
        return {"workload": "C3: Llama-2-7B-shaped prefill of a 2048-token synthetic prompt (+ first token)",
                "path": "tensor cores (tcgen05 kind::i8 signed-digit GEMMs + exact causal attention)" if tc
                        else "decode kernel (exact fallback)",
                "prompt_tokens": n_prompt, "ms": ms, "tokens_per_s": n_prompt / (ms / 1e3),
                "first_token_matches_golden": (first == gold) if gold is not None else None,
                "roofline": {"bound": "tensor", "achieved": tops, "peak": peak, "unit": "TOP/s (int8)",
                             "frac": tops / peak, "peak_kind": kind, "algorithmic_ops": ops,
                             "note": "algorithmic ops (SURVEY 8d) over the whole prefill time, CUDA-core "
                                     "attention included; the signed-digit GEMMs issue 3 MMAs per MAC"}}
    except Exception as e:
        return {"workload": "C3", "unavailable": str(e)}


def batch_c5(P, mf, cfg, dev, rank=0, n_seqs=8):
    """C5 shard of rank r: sequences 8r .. 8r+7 (prompt seed 8 for sequence
    0, 1000+i otherwise; P=16, N=128) generated together through the public
    batch call (host prompts in, host tokens + BLAKE3 hashes out), wall
    clock; every hash checked against the committed goldens
    (tests/golden/models_7b.json c5_i, C oracle pinned to the reference)."""
    try:
        ids = list(range(n_seqs * rank, n_seqs * (rank + 1)))
        prompts = [P.prompt_from_seed(8 if i == 0 else 1000 + i, cfg.vocab, 16) for i in ids]
        P.generate_greedy_batch(mf, prompts, 128, device=dev)  # warm: buffers + the captured step graph
        times = []
        for _ in range(3):
            t = time.perf_counter()
            res, path = P.generate_greedy_batch(mf, prompts, 128, device=dev)
            times.append(time.perf_counter() - t)
        dt = sorted(times)[1]
        gold = golden_c2()
        checked = [i for i in ids if f"c5_{i}" in gold]
        ok = sum(res[ids.index(i)].output_hash.hex() == gold[f"c5_{i}"]["output_hash"] for i in checked)
        return {"workload": f"C5 shard: {n_seqs} independent sequences (ids {ids[0]}..{ids[-1]}), P=16, N=128, "
                            "generated together",
                "path": path, "seconds": dt, "tokens_per_s": n_seqs * 128 / dt, "golden_checked": len(checked),
                "golden_hash_matches": ok, "mismatches": len(checked) - ok,
                "timing": "wall clock of dimg_generate_greedy_batch (prompt phase + 128 graph-replayed steps), "
                          "median of 3 after one warm call"}
    except Exception as e:
        return {"workload": "C5", "unavailable": str(e)}


def blake3_leg(P, mf, dev, peak_gbs):
    """the model-bytes hash (weight_hash, proj/src/model.cpp:310)
    on the GPU over the 6.75 GB container resident in HBM: kernel time by CUDA
    events, checked against the host hash of the same bytes."""
    try:
        import numpy as np
        import torch
        host = np.frombuffer(mf.bytes, np.uint8)
        buf = torch.from_numpy(host).to(f"cuda:{dev}")
        torch.cuda.synchronize(dev)
        P.blake3_device(buf.data_ptr(), host.size, device=dev)  # warm
        times = []
        for _ in range(3):
            got, ms = P.blake3_device(buf.data_ptr(), host.size, device=dev, timed=True)
            times.append(ms)
        ms = sorted(times)[1]
        del buf
        gbs = host.size / ms / 1e6
        return {"workload": "BLAKE3 of the 7B DIM1 container (weight_hash), device-resident",
                "bytes": int(host.size), "ms": ms, "gbs": gbs, "matches_host_hash": got.hex() == mf.weight_hash,
                "roofline": {"bound": "int ALU (ncu sm__pipe_alu_cycles_active 97%)", "hbm_frac": gbs / peak_gbs},
                "timing": "CUDA events around the four tree-hash launches, median of 3"}
    except Exception as e:
        return {"workload": "BLAKE3", "unavailable": str(e)}


def tp_one_gpu(P, mf, prompt, gold, steps):
    """The fused tensor-parallel program for g = 2, 4, 8 with every shard on
    this one GPU (backend "fused": one cooperative launch, the g ranks' CTAs
    share its SMs and HBM and exchange through device memory). Per-token time
    against the single-GPU kernel = the cost of the in-kernel exchange and of
    the narrower per-rank grids -- not a multi-GPU scaling number."""
    out = {"workload": "C2 decode, fused TP program, all g shards on one GPU", "steps": steps}
    try:
        for g in (2, 4, 8):
            tp = P.TensorParallel(mf, g, backend="fused")
            tp.time_decode(prompt, 8)
            ms = tp.time_decode(prompt, steps)
            toks = tp.tokens(steps)
            n = min(len(toks), len(gold.get("tokens", [])))
            out[f"g{g}"] = {"ms_per_step": ms / steps, "tokens_match_c2_golden": toks[:n] == gold["tokens"][:n]}
            tp.close()
    except Exception as e:  # reported, not fatal to the headline
        out["error"] = repr(e)
    return out


def run_ours(args, rank, world, local):
    import paper_2603_24904_b200 as P
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local
    cfg = P.ModelConfig(*CFG7B)
    t0 = time.time()
    mf = P.gen_toy_model(MODEL_SEED, cfg, device=dev)  # weight stream on the GPU (same bytes)
    gen_s = time.time() - t0
    wh_ok = mf.weight_hash == WEIGHT_HASH_7B if rank == 0 else None
    prompt = P.prompt_from_seed(PROMPT_SEED, cfg.vocab, PROMPT_LEN)
    gold = golden_c2().get("c2", {})
    peak, peak_kind = peaks()
    step_bytes = bytes_per_token(cfg.n_layers, cfg.d_model, cfg.d_ffn, cfg.vocab)

    def barrier():
        if dist is not None:
            dist.barrier()

    def allreduce(v, op):
        if dist is None:
            return v
        import torch
        t = torch.tensor([v], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return float(t.item())

    with ClockSampler(dev) as clk_all:
        if world == 1 and not args.tp:
            sess = P.InferenceSession(mf, P.EngineOptions(device=dev))
            n_total = args.warmup + args.steps
            sess.begin(prompt, n_total)
            sess.prefill()
            sess.decode(args.warmup)
            sess.sync()
            with ClockSampler(dev) as clk:
                ms = sess.time_decode(args.steps)  # CUDA events on the session stream, synced both sides
            toks = sess.tokens(n_total)
            launches, _ = sess.launches()
            gpu_launches = launches  # one persistent launch runs all K steps
            kernel = "decode_persistent_kernel (per decode step)"
            # e2e: the reference-shaped call with host buffers (C2: P=16, N=128)
            sess.generate_greedy(prompt, 128)  # warm
            t1 = time.perf_counter()
            for _ in range(3):
                res = sess.generate_greedy(prompt, 128)
            e2e_s = (time.perf_counter() - t1) / 3
            e2e_call = "dimg_generate_greedy(prompt 16 -> 128 tokens, BLAKE3 on host)"
            extra = {}
        else:
            # tensor parallel, fused: every rank's persistent kernel exchanges
            # the partial sums over peer memory (handles via torch.distributed).
            # A probe (construct, connect, one short decode) must succeed on
            # every rank first; otherwise every rank takes the NCCL TP path as
            # the headline (same collectives on all ranks, so none is left
            # waiting), and the line says why.
            def tp_headline(tp, backend):
                tp.time_decode(prompt, args.warmup)  # warm
                barrier()
                with ClockSampler(dev) as clk_:
                    ms_ = tp.time_decode(prompt, args.warmup + args.steps)
                    ms_w = tp.time_decode(prompt, args.warmup)
                barrier()
                # the K steps after W warm ones: difference of two CUDA-event timed launches
                ms_ = max(ms_ - ms_w, 1e-6)
                toks_ = tp.tokens(args.warmup + args.steps)
                info_ = tp.info()
                tp.generate_greedy(prompt, 128)  # warm
                barrier()
                t1_ = time.perf_counter()
                for _ in range(3):
                    res_ = tp.generate_greedy(prompt, 128)
                e2e_ = (time.perf_counter() - t1_) / 3
                return ms_, clk_, toks_, info_, res_, e2e_

            tp, fused_err = None, None
            try:
                if os.environ.get("DIMG_BENCH_FORCE_NCCL"):  # exercises the fallback
                    raise RuntimeError("DIMG_BENCH_FORCE_NCCL set")
                tp = P.TensorParallel(mf, world, backend="fused-ipc", rank=rank, device=dev)
            except Exception as e:
                fused_err = f"{type(e).__name__}: {e}"[:300]
            if world > 1 and allreduce(0.0 if fused_err else 1.0, dist.ReduceOp.MIN) < 1:
                fused_err = fused_err or "a peer rank could not build its fused-ipc shard"
            if fused_err is None:
                try:
                    if world > 1:
                        tp.connect_group()
                    tp.time_decode(prompt, 2)  # probe: one launch, in-kernel exchange with every peer
                except Exception as e:
                    fused_err = f"{type(e).__name__}: {e}"[:300]
                if world > 1 and allreduce(0.0 if fused_err else 1.0, dist.ReduceOp.MIN) < 1:
                    fused_err = fused_err or "a peer rank's fused-ipc probe failed"
            if fused_err is None:
                ms, clk, toks, info, res, e2e_s = tp_headline(tp, "fused-ipc")
                gpu_launches = 2  # the two timed persistent launches (all their steps inside)
                kernel = ("decode_persistent_kernel on the rank's shard, WO/w_down sums exchanged in-kernel "
                          "(per step, per GPU)")
                e2e_call = "dimg_tp_generate_greedy(prompt 16 -> 128 tokens, BLAKE3 on host), fused-ipc tp"
                extra = {"tp_group": {"backend": "fused-ipc", "ranks": world,
                                      "exchange": "CUDA IPC peer memory, in-kernel",
                                      "handles_gathered_over": "torch.distributed (nccl process group)",
                                      "weight_bytes_per_rank": info["weight_bytes"]}}
                tp.close()
            else:
                if tp is not None:
                    tp.close()
                obj = [P.nccl_unique_id() if rank == 0 else None]
                if world > 1:
                    dist.broadcast_object_list(obj, src=0)
                tpn = P.TensorParallel(mf, world, backend="nccl", rank=rank, nccl_id=obj[0], device=dev)
                ms, clk, toks, info, res, e2e_s = tp_headline(tpn, "nccl")
                gpu_launches = info["launches_per_step"] * (2 * args.warmup + args.steps)  # the two timed calls
                kernel = "per-stage GEMV kernels on the rank's shard + ncclAllReduce (fused-ipc fallback)"
                e2e_call = "dimg_tp_generate_greedy(prompt 16 -> 128 tokens, BLAKE3 on host), nccl tp"
                extra = {"tp_group": {"backend": "nccl", "ranks": world, "fused_ipc_error": fused_err,
                                      "weight_bytes_per_rank": info["weight_bytes"]}}
                tpn.close()
    ms_max = allreduce(ms, dist.ReduceOp.MAX if dist else None)
    e2e_s = allreduce(e2e_s, dist.ReduceOp.MAX if dist else None)
    per_step_ms = ms_max / args.steps
    value = args.steps / (ms_max / 1e3)
    n_chk = min(len(toks), len(gold.get("tokens", [])))
    tokens_ok = toks[:n_chk] == gold["tokens"][:n_chk] if n_chk else None
    gpu_bytes = step_bytes / world
    step_gbs = gpu_bytes / (per_step_ms * 1e-3) / 1e9
    traffic, traffic_src = None, None
    try:  # dram__bytes_read+write per decode step from the committed ncu capture
        for fn in ("r02_traffic.json", "r01_traffic.json"):
            pth = os.path.join(ROOT, "profiles", fn)
            if os.path.exists(pth):
                with open(pth) as f:
                    traffic = json.load(f)["traffic_bytes_per_step"]
                traffic_src = f"profiles/{fn} (ncu --set full capture of one decode step, not this run)"
                break
    except Exception:
        pass
    e2e = {"value": 128 / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": 4 * PROMPT_LEN,
           "d2h_bytes_per_step": 4 * 128, "call": e2e_call, "output_hash": res.output_hash.hex(),
           "hash_matches_c2_golden": res.output_hash.hex() == gold.get("output_hash")}

    base = cpu_baseline(mf, CFG7B) if (rank == 0 and world == 1 and not args.no_cpu_baseline) else None
    legs = not args.no_prefill
    prefill = prefill_c3(P, mf, cfg, dev) if rank == 0 and legs else None
    batch = batch_c5(P, mf, cfg, dev, rank=rank) if legs else None
    blake3 = blake3_leg(P, mf, dev, peak) if rank == 0 and legs and world == 1 else None
    c5 = dp = None
    if world > 1 and legs:
        # C5 across the ranks: 8 sequences each, hashes vs the goldens
        n_ok = allreduce(float(batch.get("golden_hash_matches", 0) or 0), dist.ReduceOp.SUM)
        n_chk = allreduce(float(batch.get("golden_checked", 0) or 0), dist.ReduceOp.SUM)
        t_max = allreduce(float(batch.get("seconds", 0) or 0), dist.ReduceOp.MAX)
        c5 = {"workload": f"C5: {8 * world} independent sequences, 8 per GPU, P=16, N=128",
              "tokens_per_s": 8 * world * 128 / t_max if t_max else None, "seconds_max_over_ranks": t_max,
              "golden_checked": int(n_chk), "golden_hash_matches": int(n_ok), "mismatches": int(n_chk - n_ok),
              "rank0": batch}
        # weak-scaling replicas: every rank its own sequence on the single-GPU kernel
        sess = P.InferenceSession(mf, P.EngineOptions(device=dev))
        pseed = PROMPT_SEED if rank == 0 else 1000 + rank
        sess.begin(P.prompt_from_seed(pseed, cfg.vocab, PROMPT_LEN), args.warmup + args.steps)
        sess.prefill()
        sess.decode(args.warmup)
        sess.sync()
        barrier()
        dms = allreduce(sess.time_decode(args.steps), dist.ReduceOp.MAX)
        dp = {"workload": f"{world} independent batch-1 sequences, one per GPU (persistent kernel)",
              "tokens_per_s": world * args.steps / (dms / 1e3), "ms_per_step": dms / args.steps}
    tp_nccl = tp_one = None
    if world > 1 and legs:
        # the collective-library baseline of the same TP decode: per-stage
        # GEMVs + ncclAllReduce (rank 0 makes the NCCL id)
        obj = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        tpn = P.TensorParallel(mf, world, backend="nccl", rank=rank, nccl_id=obj[0], device=dev)
        tpn.time_decode(prompt, args.warmup)
        barrier()
        nms = tpn.time_decode(prompt, args.warmup + args.steps) - tpn.time_decode(prompt, args.warmup)
        nms = allreduce(max(nms, 1e-6), dist.ReduceOp.MAX)
        ntok = tpn.tokens(args.warmup + args.steps)
        nn = min(len(ntok), len(gold.get("tokens", [])))
        tp_nccl = {"workload": f"C4/C2 tensor parallel tp{world}: per-stage GEMVs + ncclAllReduce",
                   "tokens_per_s": args.steps / (nms / 1e3), "ms_per_step": nms / args.steps,
                   "launches_per_step": tpn.info()["launches_per_step"], "nccl_comm_init": "ncclCommInitRank",
                   "tokens_match_c2_golden": ntok[:nn] == gold["tokens"][:nn] if nn else None}
        tpn.close()
    if world == 1 and rank == 0 and legs:
        tp_one = tp_one_gpu(P, mf, prompt, gold, args.steps)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step_ms,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "int64",
            "data": "synthetic (gen_toy_model seed 7: uniform int8 weights, Q16 scales; ChaCha20 prompt)",
            "config": config_dict(world, {"weight_hash_ok": wh_ok, "model_gen_s": round(gen_s, 1)}),
            "tokens_match_c2_golden": tokens_ok,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "roofline": {"bound": "hbm", "achieved": step_gbs, "peak": peak, "unit": "GB/s",
                         "frac": step_gbs / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": kernel, "bytes_per_step_per_gpu": gpu_bytes, "ms_per_step": per_step_ms,
                         "peak_kind": peak_kind},
            "clocks": dict(clk.summary(), whole_run=clk_all.summary()),
            "cpu_baseline": base,
            "prefill": prefill,
            "batch": batch if world == 1 else None,
            "c5": c5,
            "dp": dp,
            "tp_nccl": tp_nccl,
            "tp_one_gpu": tp_one,
            "blake3": blake3,
            "tokens_head": toks[:8],
        }
        line.update(extra)
        emit(line)
    if dist is not None:
        dist.destroy_process_group()
    return 0


_JSON_FD = None


def emit(line):
    """The one JSON line, on the process's original stdout."""
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    global _JSON_FD
    # everything but the JSON line goes to stderr: libraries print to fd 1
    # (NCCL's version banner at communicator init, for one)
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--no-prefill", action="store_true", help="skip the C3 prefill and C5 batch measurements")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tp", action="store_true", help="the tensor-parallel (NCCL) path even at N = 1 (tests)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank, world, local = env_rank()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
