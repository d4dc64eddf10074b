#!/usr/bin/env python3
"""Benchmark: decode tokens/s of the Llama-2-7B-shaped integer model (BASELINE.json
configs[1]: 7B-shaped random-init int8 weights, seed 7; ChaCha20 prompt seed 8,
16 tokens; batch-1 greedy decode) on N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one greedy decode token: one full forward of the 32-layer model
(6.62 GB of int8 weights + scales streamed from HBM) plus the on-device
argmax that appends the next token. With N > 1 (torchrun, one process per
GPU) every rank decodes its own independent sequence (weak scaling, no
data-path collective; C5's sequence sharding): value = all ranks' tokens /
max-over-ranks time.

Keys beyond the base contract:
  e2e           the same metric through the reference-shaped C-ABI call
                dimg_generate_greedy with HOST buffers (prompt H2D, tokens D2H
                and the BLAKE3 hash inside the timed region)
  roofline      dominant kernel (gate/up GEMV): algorithmic bytes per launch /
                CUDA-event launch time, vs MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the reference engine (oracle/_ref, compiled from its own
                sources) timed on this host, rank 0, N=1
--impl reference times that reference engine alone on the same workload.
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


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        mx = max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------------------
def reference_model(ref, cfg):
    """The reference's own gen_toy_model (proj/src/model.cpp:189-215)."""
    return ref.gen_toy(MODEL_SEED, cfg)


def time_reference(ref, m, n_warm, n_timed, prompt, threads):
    """Greedy decode through dim::InferenceSession::forward (+select_greedy),
    the reference's stock path. Returns seconds per decode forward."""
    import ctypes as C

    import numpy as np
    h = C.c_void_p()
    assert ref.lib.ref_session_new(m.h, threads, C.byref(h)) == 0
    nxt = C.c_uint32()
    pos = 0
    for t in prompt:  # prefill sample (untimed)
        assert ref.lib.ref_session_forward(h, int(t), pos, None, C.byref(nxt)) == 0
        pos += 1
    for _ in range(n_warm):
        assert ref.lib.ref_session_forward(h, nxt.value, pos, None, C.byref(nxt)) == 0
        pos += 1
    t0 = time.perf_counter()
    for _ in range(n_timed):
        assert ref.lib.ref_session_forward(h, nxt.value, pos, None, C.byref(nxt)) == 0
        pos += 1
    dt = time.perf_counter() - t0
    ref.lib.ref_session_free(h)
    del np
    return dt / max(1, n_timed)


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from oracle.pyoracle import Config, Reference
    cfg = Config(*CFG7B)
    threads = os.cpu_count() or 1
    if not Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libdimref.so not built"}))
        return 0
    ref = Reference()
    t0 = time.time()
    m = reference_model(ref, cfg)
    gen_s = time.time() - t0
    prompt = ref.prompt(PROMPT_SEED, cfg.vocab, PROMPT_LEN)[:4]
    spf = time_reference(ref, m, args.warmup, args.steps, prompt, threads)
    value = 1.0 / spf
    sample = (f"dim::InferenceSession::forward + select_greedy, {args.steps} timed decode "
              f"forwards after a 4-token prompt and {args.warmup} warm-up forwards "
              f"(threads={threads}: the reference's dense matvec is single-threaded)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": spf * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic (reference gen_toy_model seed 7)",
        "config": {"workload": "C2: Llama-2-7B-shaped int8/Q16 model, batch-1 greedy decode",
                   "model": "llama2-7b-shaped-int", "seed": MODEL_SEED, "prompt_seed": PROMPT_SEED},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": 1, "kind": "reference",
                         "sample": sample, "threads_setting": threads, "model_gen_s": round(gen_s, 1)},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
def cpu_baseline(model_file, cfg_t):
    """Reference engine on this host over the SAME weights (bounded sample)."""
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
        spf = time_reference(ref, m, 0, 3, prompt, 1)
        return {"value": 1.0 / spf, "unit": "tokens/s", "cores": 1, "kind": "reference",
                "sample": "3 decode forwards (dim::InferenceSession::forward + select_greedy) after a "
                          "2-token prompt, same weights, threads=1"}
    except Exception as e:  # reported, never fatal for the GPU number
        return {"value": None, "unit": "tokens/s", "cores": 1, "kind": "reference",
                "sample": f"unavailable: {e}"}


def prefill_c3(P, mf, cfg, dev):
    """C3: prefill of a 2048-token synthetic prompt (prompt seed 9) on the
    tensor cores, timed with CUDA events (2 warm + 3 timed); the positions
    0..2046 go through every layer, the last prompt token is the first decode
    step. Roofline: int8 tensor ops of the limb GEMMs (3 limbs per dense MAC)
    against 2 x the measured bf16 peak (kind::i8 issues at twice kind::f16)."""
    try:
        n_prompt = 2048
        prompt = P.prompt_from_seed(9, cfg.vocab, n_prompt)
        s = P.InferenceSession(mf, P.EngineOptions(device=dev))
        times, tc = [], True
        for i in range(5):
            s.begin(prompt, 1)
            ms, used = s.time_prefill()
            tc &= used
            if i >= 2:
                times.append(ms)
        ms = sorted(times)[len(times) // 2]
        n = n_prompt - 1
        D, F, L = cfg.d_model, cfg.d_ffn, cfg.n_layers
        macs = n * ((L - 1) * (4 * D * D + 3 * F * D) + 3 * D * D)
        limb_ops = 2 * 3 * macs
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                peak = 2 * json.load(f)["bf16_tflops"]
            kind = "2 x measured bf16 burst (kind::i8 at twice the kind::f16 rate)"
        except Exception:
            peak, kind = 2 * 1590.0, "2 x fallback bf16"
        return {"workload": "C3: Llama-2-7B-shaped prefill of a 2048-token synthetic prompt",
                "path": "tensor cores (tcgen05 kind::i8 limb GEMMs + exact causal attention)" if tc
                        else "decode kernel (exact fallback)",
                "prompt_tokens": n_prompt, "positions_prefilled": n, "ms": ms,
                "tokens_per_s": n / (ms / 1e3),
                "roofline_whole_prefill": {"bound": "tensor", "achieved": limb_ops / (ms / 1e3) / 1e12,
                                           "peak": peak, "unit": "TOP/s (int8)",
                                           "frac": limb_ops / (ms / 1e3) / 1e12 / peak, "peak_kind": kind,
                                           "note": "whole prefill time incl. the CUDA-core attention "
                                                   "(profiles/r01_prefill_launches.txt has the split)"}}
    except Exception as e:
        return {"workload": "C3", "unavailable": str(e)}


def batch_c5(P, mf, cfg, dev, n_seqs=8):
    """C5 on this GPU: n_seqs independent sequences (prompt seeds 8, 1001,
    ...; P=16, N=128) generated together through the public batch call
    (host prompts in, host tokens + BLAKE3 hashes out), wall-clock; hashes
    checked against the committed goldens (tests/golden/models_7b.json)."""
    try:
        prompts = [P.prompt_from_seed(8 if i == 0 else 1000 + i, cfg.vocab, 16) for i in range(n_seqs)]
        P.generate_greedy_batch(mf, prompts, 128, device=dev)  # warm: buffers + the captured step graph
        times = []
        for _ in range(3):
            t = time.perf_counter()
            res, path = P.generate_greedy_batch(mf, prompts, 128, device=dev)
            times.append(time.perf_counter() - t)
        dt = sorted(times)[1]
        ok = None
        try:
            with open(os.path.join(ROOT, "tests", "golden", "models_7b.json")) as f:
                gold = json.load(f)
            ok = sum(res[i].output_hash.hex() == gold[f"c5_{i}"]["output_hash"] for i in range(n_seqs)
                     if f"c5_{i}" in gold)
        except Exception:
            pass
        return {"workload": f"C5 shard: {n_seqs} independent sequences, P=16, N=128, generated together",
                "path": path, "seconds": dt, "tokens_per_s": n_seqs * 128 / dt, "golden_hash_matches": ok,
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


def run_ours(args, rank, world, local):
    import numpy as np

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
    wh_ok = None
    if rank == 0:
        wh_ok = mf.weight_hash == WEIGHT_HASH_7B
    # rank r decodes its own sequence: C5's prompt seeds (8, then 1000+r)
    pseed = PROMPT_SEED if rank == 0 else 1000 + rank
    prompt = P.prompt_from_seed(pseed, cfg.vocab, PROMPT_LEN)
    sess = P.InferenceSession(mf, P.EngineOptions(device=dev))
    n_total = args.warmup + args.steps
    sess.begin(prompt, n_total)
    sess.prefill()
    sess.decode(args.warmup)
    sess.sync()

    def barrier():
        if dist is not None:
            dist.barrier()

    barrier()
    with ClockSampler(dev) as clk:
        ms = sess.time_decode(args.steps)  # CUDA events on the session stream, synced both sides
    barrier()
    ms_max = ms
    if dist is not None:
        import torch
        t = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    toks = sess.tokens(n_total)
    per_step_ms = ms_max / args.steps
    value = world * args.steps / (ms_max / 1e3)
    launches_per_step, _ = sess.launches()

    # per-stage probes (each stage kind replayed over the layers in one launch)
    kern = {}
    for which, name in enumerate(sess.KERNELS):
        kms, kb = sess.time_kernel(which, 64 if which != 4 else 16)
        kern[name] = {"ms": kms, "bytes": kb, "gbs": kb / (kms * 1e-3) / 1e9}
    peak, peak_kind = peaks()
    step_bytes = bytes_per_token(cfg.n_layers, cfg.d_model, cfg.d_ffn, cfg.vocab)
    step_gbs = step_bytes / (per_step_ms * 1e-3) / 1e9
    traffic = None
    try:  # dram__bytes_read+write per decode step from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as f:
            traffic = json.load(f)["traffic_bytes_per_step"]
    except Exception:
        pass

    # e2e: the reference-shaped call with host buffers (C2: P=16, N=128)
    e2e = None
    if rank == 0 or world > 1:
        n_new = 128
        sess.generate_greedy(prompt, n_new)  # warm
        reps = 3
        t1 = time.perf_counter()
        for _ in range(reps):
            res = sess.generate_greedy(prompt, n_new)
        e2e_s = (time.perf_counter() - t1) / reps
        e2e = {"value": n_new / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": 4 * PROMPT_LEN,
               "d2h_bytes_per_step": 4 * n_new,
               "call": "dimg_generate_greedy(prompt 16 -> 128 tokens, BLAKE3 on host)",
               "output_hash": res.output_hash.hex()}
    if dist is not None:
        import torch
        t = torch.tensor([e2e["value"] if e2e else 0.0], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if e2e:
            e2e["value"] = float(t.item()) * world
    base = cpu_baseline(mf, CFG7B) if (rank == 0 and world == 1 and not args.no_cpu_baseline) else None
    prefill = prefill_c3(P, mf, cfg, dev) if rank == 0 and not args.no_prefill else None
    batch = batch_c5(P, mf, cfg, dev) if rank == 0 and not args.no_prefill else None
    blake3 = blake3_leg(P, mf, dev, peak) if rank == 0 and not args.no_prefill else None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (gen_toy_model seed 7: uniform int8 weights, Q16 scales; ChaCha20 prompt)",
            "config": {"workload": "C2: Llama-2-7B-shaped int8/Q16 model, batch-1 greedy decode",
                       "model": "llama2-7b-shaped-int", "layers": cfg.n_layers,
                       "d_model": cfg.d_model, "d_ffn": cfg.d_ffn, "vocab": cfg.vocab,
                       "seed": MODEL_SEED, "prompt_seed": PROMPT_SEED, "prompt_len": PROMPT_LEN,
                       "global_batch": world, "parallelism": f"dp{world} (independent sequences)",
                       "l2": "weights 6.6 GB/step > 126 MB L2 (no flush needed)",
                       "weight_hash_ok": wh_ok, "model_gen_s": round(gen_s, 1)},
            "e2e": e2e,
            "gpu_launches": launches_per_step,  # one persistent launch runs all K steps
            # dominant kernel: the persistent decode kernel (99.8% of GPU time,
            # profiles/r01_bench_launches.csv); one decode step = 6.62 GB of
            # algorithmic weight bytes, timed with CUDA events on its stream
            "roofline": {"bound": "hbm", "achieved": step_gbs, "peak": peak, "unit": "GB/s",
                         "frac": step_gbs / peak, "traffic": traffic,
                         "kernel": "decode_persistent_kernel (per decode step)",
                         "bytes_per_step": step_bytes, "ms_per_step": per_step_ms,
                         "peak_kind": peak_kind},
            "stages": kern,
            "clocks": clk.summary(),
            "cpu_baseline": base,
            "prefill": prefill,
            "batch": batch,
            "blake3": blake3,
            "tokens_head": toks[:8],
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--no-prefill", action="store_true", help="skip the C3 prefill and C5 batch measurements")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank, world, local = env_rank()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
