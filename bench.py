"""Benchmark: COMET-22 (XLM-R-large-shaped) segment scoring on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--precision fp32]
    python bench.py --impl reference ...      # the reference algorithm on host cores

One step = one maxi-batch window of 1024 records (mini_batch 128 x factor 8,
the reference Evaluator's default window, `pkg/src/metricforge/evaluate.py:168-177`)
of synthetic wmt22-comet-da-shaped triplets (content length
~U{1..126} per field, one id per word, N(0, 0.02^2) random-init weights).

  value   records/s over K steps with the packed token ids already resident in
          HBM (mfg_score_device), CUDA events on the stream libmfgpu launches on,
          max over ranks.
  e2e     the same metric through the public API: Evaluator.evaluate_lines on
          host TSV text (tokenisation, plan, packing, H2D, device, D2H, order
          restore), wall clock with device syncs, max over ranks.
  roofline  dominant kernel class (a tcgen05 GEMM) from per-launch CUDA events
          in the timed region: algorithmic FLOPs per launch / mean duration vs
          the measured sustained bf16 peak (MEASURED_PEAKS.json).
  cpu_baseline  the reference algorithm (oracle numpy port) on the host cores,
          bounded sample of the same workload, rank 0 at N=1 only.

Multi-GPU (torchrun): one rank per GPU, each scores its own windows (records
are independent; no collective on the data path), barrier + max-over-ranks
timing; scaling "weak".
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "COMET-22 segments/sec at 1/2/4/8 B200; GEMM tensor-pipe util vs peak"
UNIT = "segments/s"
RECORDS_PER_STEP = 1024
BENCH_DIR = os.environ.get("MFG_BENCH_DIR", "/tmp/mfg_bench")


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# --------------------------------------------------------------------------- helpers
def prepare_model(cfg, rank, world, barrier):
    """Synthetic container + vocab for config `cfg` (written once per box)."""
    from oracle import fixtures as fx
    from paper_2408_11853_b200.container import ModelManifest, write_container

    os.makedirs(BENCH_DIR, exist_ok=True)
    man = dict(fx.CONFIGS[cfg])
    path = os.path.join(BENCH_DIR, f"config{cfg}.mfrg")
    vocab = os.path.join(BENCH_DIR, f"config{cfg}.vocab.txt")
    done = path + ".ok"
    if env_int("LOCAL_RANK", 0) == 0 and not os.path.exists(done):
        if cfg == 1:  # the reference fixture family (std-0.25 weights, 64-token vocab)
            w = fx.fixture_weights(man, 1234)
            tensors = [(n, "f32", w[n].shape, w[n]) for n, _ in fx.tensor_shapes(man)]
            fx.write_vocab(vocab, fx.fixture_vocab_lines())
        else:
            tensors = ((n, "f32", a.shape, a) for n, a in fx.synthetic_weights(man))
            fx.write_vocab(vocab, fx.synthetic_vocab_lines(man["vocab_size"]))
        write_container(ModelManifest(**man), tensors, path)
        open(done, "w").close()
    barrier()
    while not os.path.exists(done):
        time.sleep(0.5)
    return man, path, vocab


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def ncu_traffic(cls=None):
    """dram bytes per launch of kernel class `cls` (else the dominant GEMM) from the
    newest committed ncu summary (profiles/ncu_summary_*.json)."""
    for name in sorted(os.listdir(os.path.join(ROOT, "profiles")), reverse=True) \
            if os.path.isdir(os.path.join(ROOT, "profiles")) else []:
        if name.startswith("ncu_summary") and name.endswith(".json"):
            try:
                with open(os.path.join(ROOT, "profiles", name)) as f:
                    summ = json.load(f)
                if cls and cls in summ.get("by_class", {}):
                    return summ["by_class"][cls]["dram_bytes"], name
                return summ.get("dram_bytes_per_launch"), name
            except Exception:
                pass
    return None, None


def workload_lines(cfg, n, seed):
    from oracle import fixtures as fx
    if cfg == 1:
        return fx.fixture_tsv_lines("comet", n, seed=seed)
    return fx.synthetic_tsv_lines(cfg, n, seed=seed)


def oracle_model(cfg):
    from oracle import fixtures as fx
    from oracle import tokenizer as otk
    from oracle.encoder import OracleModel
    man = dict(fx.CONFIGS[cfg])
    if cfg == 1:
        return OracleModel(man, fx.fixture_weights(man, 1234)), otk.OracleVocab(fx.fixture_vocab_lines())
    return (OracleModel(man, dict(fx.synthetic_weights(man))),
            otk.OracleVocab(fx.synthetic_vocab_lines(man["vocab_size"])))


def cpu_baseline(cfg, n_records, return_scores=False):
    """Reference algorithm (oracle numpy port) on host cores, bounded sample."""
    from oracle import evaluate as oe
    from oracle import fixtures as fx
    from oracle import tokenizer as otk
    from oracle.encoder import OracleModel

    model, vocab = oracle_model(cfg)
    lines = workload_lines(cfg, n_records, fx.TEXT_SEED + 777)
    oe.score_lines(model, vocab, lines[:1])  # discard run (BLAS warmup)
    t0 = time.perf_counter()
    ref_scores, _ = oe.score_lines(model, vocab, lines)
    dt = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        cores = max((p.get("num_threads", 1) for p in threadpool_info()), default=1)
    except Exception:
        cores = os.cpu_count() or 1
    out = {"value": n_records / dt, "unit": UNIT, "cores": int(cores), "kind": "port",
           "sample": f"{n_records} synthetic config-{cfg} records (oracle numpy port of "
                     f"pkg/src/metricforge/encoder.py, fp32, {dt:.1f} s)"}
    return (out, lines, ref_scores) if return_scores else out


def parity_report(path, vocab_path, lines, ref, device, cfg_id):
    """Same records through the device path at every precision vs the fp32
    oracle (the reference algorithm): max/mean |delta| and Pearson; the fp16
    mode also against the oracle's fp16 mode (the reference's binary16 path)."""
    import paper_2408_11853_b200 as mf
    from oracle import evaluate as oe
    from oracle.encoder import OracleModel

    ref = np.asarray(ref, dtype=np.float64)
    out = {"n_records": len(lines), "tolerance": 1e-3, "reference": "oracle fp32 (numpy port)"}

    def stats(got, want):
        d = np.abs(got - want)
        pear = float(np.corrcoef(got, want)[0, 1]) if len(got) > 2 and want.std() > 0 else None
        return {"max_abs": float(d.max()), "mean_abs": float(d.mean()), "pearson": pear}

    for prec in ("fp32", "bf16x3", "bf16", "fp16"):
        cfg = mf.EvaluatorConfig(model=path, vocab=vocab_path, quiet=True, validate=False,
                                 device=device, precision=prec)
        with mf.Evaluator(cfg) as ev:
            got = np.asarray(ev.evaluate_lines(lines).segment_scores, dtype=np.float64)
        out[prec] = stats(got, ref)
        if prec == "fp16":
            model32, vocab = oracle_model(cfg_id)
            m16 = OracleModel(model32.m, {k: v for k, v in model32.w.items()}, mode="fp16")
            want16, _ = oe.score_lines(m16, vocab, lines)
            out["fp16"]["vs_reference_fp16_mode"] = stats(got, np.asarray(want16, np.float64))
    out["fp32_within_tolerance"] = out["fp32"]["max_abs"] <= 1e-3
    return out


# --------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    per_step = 2 if args.config >= 2 else 64
    base = cpu_baseline(args.config, per_step)  # also warms BLAS
    from oracle import evaluate as oe
    from oracle import fixtures as fx
    from oracle import tokenizer as otk
    from oracle.encoder import OracleModel

    model, vocab = oracle_model(args.config)
    lines = workload_lines(args.config, per_step * (args.steps + args.warmup), fx.TEXT_SEED)
    chunks = [lines[i * per_step:(i + 1) * per_step] for i in range(args.steps + args.warmup)]
    for c in chunks[:args.warmup]:
        oe.score_lines(model, vocab, c)
    t0 = time.perf_counter()
    for c in chunks[args.warmup:]:
        oe.score_lines(model, vocab, c)
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    base.update(value=value, sample=f"{per_step} records per step x {args.steps} steps (oracle "
                                    f"numpy port of the reference encoder, fp32)")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"config {args.config}: " + fx.CONFIG_NAMES[args.config],
                       "records_per_step": per_step},
            "cpu_baseline": base,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2408_11853_b200 as mf
    from oracle import fixtures as fx
    from paper_2408_11853_b200.batching import pack_roles, plan_order

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)

    def barrier():
        if world > 1:
            dist.barrier()

    man, path, vocab_path = prepare_model(args.config, rank, world, barrier)
    n_steps = args.steps + args.warmup
    R = args.records_per_step
    lines = workload_lines(args.config, R * n_steps, fx.TEXT_SEED + 1000 * rank)

    # ---------------- device-resident timing (value)
    t_load = time.perf_counter()
    model = mf.GpuScoringModel(path, device=local_rank, precision=args.precision,
                               profile=True)
    torch.cuda.synchronize()
    load_s = time.perf_counter() - t_load
    vocab = mf.load_vocab(vocab_path)
    kind = mf.Kind.parse(man["like"])
    max_len = min(512, man["max_position"])
    n_seq = mf.kinds.N_SEQUENCES[kind]
    steps = []
    tokens_per_step = []
    for s in range(n_steps):
        chunk = lines[s * R:(s + 1) * R]
        recs = list(mf.records_from_tsv_lines(chunk, kind))
        ids, off = vocab.encode_batch(kind, [r.field_values(kind) for r in recs], max_len)
        lengths = np.diff(off).reshape(R, n_seq).sum(1)
        order = plan_order(lengths, mf.BatchConfig())
        packed, cu = pack_roles(ids, off, n_seq, order)
        steps.append((torch.from_numpy(packed).to(dev), cu))
        tokens_per_step.append(int(cu[-1]))
    out = torch.empty(R, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    model.set_stream(stream.cuda_stream)
    for s in range(args.warmup):
        model.score_device(steps[s][0].data_ptr(), steps[s][1], R, out.data_ptr())
    torch.cuda.synchronize()
    model.reset_stats()
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)

    def timed_region():
        with ClockSampler(local_rank) as c:
            ev0.record(stream)
            for s in range(args.warmup, n_steps):
                model.score_device(steps[s][0].data_ptr(), steps[s][1], R, out.data_ptr())
            ev1.record(stream)
            torch.cuda.synchronize()
        barrier()
        return ev0.elapsed_time(ev1), c

    ms, clk = timed_region()
    # a run that saw hardware / thermal slowdown is re-measured once (decided
    # jointly so every rank runs the same number of timed regions)
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    flag = torch.tensor([1.0 if bad & set(clk.summary()["reasons"]) else 0.0],
                        device="cpu" if dist.is_initialized() and dist.get_backend() == "gloo" else dev)
    if world > 1:
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
    remeasured = bool(flag.item())
    if remeasured:
        model.reset_stats()
        ms, clk = timed_region()
    stats = model.stats()
    model.set_stream(0)
    model.close()

    # ---------------- the other device precisions, same inputs (reported beside value)
    others = {}
    if world == 1 and not args.no_other_precisions:
        for prec in ("fp16", "bf16", "fp32"):
            if prec == args.precision:
                continue
            m2 = mf.GpuScoringModel(path, device=local_rank, precision=prec)
            m2.set_stream(stream.cuda_stream)
            for s in range(min(args.warmup, 2)):
                m2.score_device(steps[s][0].data_ptr(), steps[s][1], R, out.data_ptr())
            k2 = min(args.steps, 6)
            torch.cuda.synchronize()
            ev0.record(stream)
            for s in range(args.warmup, args.warmup + k2):
                m2.score_device(steps[s][0].data_ptr(), steps[s][1], R, out.data_ptr())
            ev1.record(stream)
            torch.cuda.synchronize()
            ms2 = ev0.elapsed_time(ev1)
            m2.set_stream(0)
            m2.close()
            others[prec] = {"value": R * k2 / (ms2 / 1000.0), "unit": UNIT, "steps": k2,
                            "ms_per_step": ms2 / k2}
    del steps

    # ---------------- end to end through the public API (e2e)
    cfg = mf.EvaluatorConfig(model=path, vocab=vocab_path, quiet=True, validate=False,
                             device=local_rank, precision=args.precision)
    with mf.Evaluator(cfg) as ev:
        ev.evaluate_lines(lines[:R * args.warmup])
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        rep = ev.evaluate_lines(lines[R * args.warmup:])
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        e2e_stats = ev.model.stats()
    barrier()
    assert len(rep.segment_scores) == R * args.steps
    assert all(math.isfinite(v) for v in rep.segment_scores)

    # ---------------- reduce over ranks
    vals = torch.tensor([ms, e2e_s], dtype=torch.float64,
                        device="cpu" if dist.is_initialized() and dist.get_backend() == "gloo" else dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms_max, e2e_max = float(vals[0]), float(vals[1])
    if rank != 0:
        return
    total = R * args.steps * world
    value = total / (ms_max / 1000.0)
    e2e_value = total / e2e_max

    peaks, peak_src = measured_peaks()
    cls = stats["classes"]
    gemm_names = ("qkv", "o_proj", "ffn1", "ffn2")
    dom = max(gemm_names, key=lambda k: cls[k]["ms"])
    c = cls[dom]
    per_launch_ms = c["ms"] / max(1, c["launches"])
    achieved = (c["flops"] / max(1, c["launches"])) / (per_launch_ms / 1e3) / 1e12
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
    mma_per_step = 1 if args.precision in ("bf16", "fp16") else 3
    traffic, traffic_src = ncu_traffic(dom)
    gemm_ms = sum(cls[k]["ms"] for k in gemm_names)
    gemm_flops = sum(cls[k]["flops"] for k in gemm_names)
    all_ms = sum(v["ms"] for v in cls.values())
    roofline = {
        "bound": "tensor", "kernel": f"gemm_tc_kernel ({dom})", "achieved": achieved,
        "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
        "peak_source": f"{peak_src} bf16_tflops_sustained (kernel timed inside a long step)",
        "algorithmic_flops_per_launch": c["flops"] / max(1, c["launches"]),
        "mean_launch_ms": per_launch_ms,
        "issued_mma_per_algorithmic": mma_per_step,
        "issued_frac": achieved * mma_per_step / peak,
        "all_gemms": {"achieved_tflops": gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms else None,
                      "share_of_step": gemm_ms / all_ms if all_ms else None},
        "class_ms_share": {k: v["ms"] / all_ms for k, v in cls.items()} if all_ms else {},
        "traffic_source": traffic_src,
    }
    if cls["attention"]["ms"]:
        gbs = cls["attention"]["bytes"] / (cls["attention"]["ms"] / 1e3) / 1e9
        att_traffic, _ = ncu_traffic("attention")
        roofline["attention_hbm"] = {
            "achieved_gbs": gbs, "peak_gbs": peaks.get("hbm_gbs"),
            "frac": gbs / peaks.get("hbm_gbs", 6544.3),
            "algorithmic_bytes_per_launch": cls["attention"]["bytes"] / max(1, cls["attention"]["launches"]),
            "traffic": att_traffic,
            "tflops": cls["attention"]["flops"] / (cls["attention"]["ms"] / 1e3) / 1e12}
    if cls["layernorm"]["ms"]:
        gbs = cls["layernorm"]["bytes"] / (cls["layernorm"]["ms"] / 1e3) / 1e9
        roofline["layernorm_hbm"] = {"achieved_gbs": gbs, "peak_gbs": peaks.get("hbm_gbs"),
                                     "frac": gbs / peaks.get("hbm_gbs", 6544.3)}
    h2d = sum(tokens_per_step[args.warmup:]) * 4 / args.steps + (3 * R + 1) * 4 + 8 * (
        sum(tokens_per_step[args.warmup:]) / args.steps / 64 + 3 * R)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": {"fp32": "fp16x3-split (fp32-parity)", "bf16x3": "bf16x3-split",
                  "bf16": "bf16", "fp16": "fp16 (reference binary16 mode)"}[args.precision],
        "data": ("synthetic (reference fixture generator, std-0.25 fixture weights)" if args.config == 1
                 else "synthetic (SURVEY §8d generator; random-init N(0,0.02) weights)"),
        "config": {"workload": f"config {args.config}: " + fx.CONFIG_NAMES[args.config],
                   "model": "XLM-R-large-shaped encoder (24 x d1024 x h16 x ffn4096) + "
                            "head [6144,3072,1024,1]" if args.config == 2 else fx.CONFIG_NAMES[args.config],
                   "records_per_step": R, "tokens_per_step": sum(tokens_per_step[args.warmup:]) / args.steps,
                   "precision": args.precision, "parallelism": f"dp{world} (records sharded)",
                   "l2": "inputs larger than L2 ({:.1f} GB of layer weights + GB-scale activations "
                         "per step)".format(man["n_layers"] * (4 * man["d_model"] ** 2 + 2 * man["d_model"]
                                                               * man["d_ffn"]) *
                                            (4 if args.precision in ("fp32", "bf16x3") else 2) / 1e9)},
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": R * 4 + 4,
                "path": "Evaluator.evaluate_lines (host TSV -> libmfhost -> libmfgpu -> scores)"},
        "gpu_launches": int(stats["kernel_launches"]),
        "other_precisions": others,
        "model_load_s": load_s,
        "clocks": dict(clk.summary(), remeasured=remeasured),
    }
    if world == 1 and not args.no_cpu_baseline:
        n_cpu = args.cpu_records or {1: 1024, 5: 4}.get(args.config, 8)
        base, ref_lines, ref = cpu_baseline(args.config, n_cpu, return_scores=True)
        line["cpu_baseline"] = base
        line["parity"] = parity_report(path, vocab_path, ref_lines, ref, local_rank, args.config)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "bf16x3", "bf16", "fp16"])
    ap.add_argument("--records-per-step", type=int, default=RECORDS_PER_STEP)
    ap.add_argument("--cpu-records", type=int, default=None,
                    help="CPU-baseline / parity sample (default: 1024 at config 1, 4 at config 5, "
                         "else 8 records: ~5-30 s of host work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-precisions", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    # MFG_BENCH_BACKEND=gloo: code-path check of the multi-rank bench on a box with
    # fewer GPUs than ranks (ranks share devices; not a measurement)
    backend = os.environ.get("MFG_BENCH_BACKEND", "nccl")
    if world > 1:
        import torch
        import torch.distributed as dist
        if backend == "gloo":
            local_rank %= torch.cuda.device_count()
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
