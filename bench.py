"""Benchmark of the B200 CKKS engine (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--config train|ks|bootstrap|bootstrap_full|predict|ovr]
                    [--impl ours|reference]

Workloads (BASELINE.json configs):
  train      cfg4: one encrypted-LR minibatch at N=2^16 (P16 preset): 16
             ciphertexts x 32 rows of 768-d synthetic embeddings, batched
             gradient + Nesterov update + sparse-1024 bootstrap of w and u.
             metric: encrypted LR train samples/sec (whole job).
  bootstrap  cfg3: one sparse-1024 bootstrap at N=2^16.  metric: ms.
  ks         cfg2: NTT/iNTT + relinearisation key switch of 64 ciphertexts at
             the full P16 chain.  metric: key switches/sec.
  bootstrap_full  cfg3 full-slot (ingest) bootstrap, batched.  metric: ms/ct.
  predict    cfg1: P14 encrypt -> 768-d inference -> decrypt.  metric: ms.
  ovr        cfg5: one One-vs-Rest minibatch of 4 class-models on 1024-d
             embeddings (32 ciphertexts x 16 rows), each class's update and
             sparse-2048 refresh.  metric: samples/sec (4 class-models).
--impl reference times the reference algorithm's CPU path (the oracle port,
oracle/, C+OpenMP kernels, all host cores) on a bounded sample.
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("BENCH_CONFIG", "train"))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--profile", action="store_true", help="print per-kernel-class profile")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------


def init_dist(args):
    import torch

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1:
        import torch.distributed as dist

        # BENCH_ONE_DEVICE_GLOO=1: every rank on cuda:0 over gloo -- a functional
        # check of the multi-rank path on a one-GPU box (NCCL refuses two ranks
        # on one device); its timings are not a scaling measurement
        if os.environ.get("BENCH_ONE_DEVICE_GLOO") == "1":
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# clocks (sampled with nvidia-smi during the timed region)
# ---------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self):
        """NVML queries take microseconds (an nvidia-smi process ~100 ms), so
        even a sub-second timed region gets many samples.  Same row format."""
        import pynvml as nv

        nv.nvmlInit()
        try:
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
            self._ready.set()  # NVML is up: sampling starts with the timed region
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(smax), ""] +
                                    ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(0.02)
        finally:
            nv.nvmlShutdown()

    def _run(self):
        try:
            return self._run_nvml()
        except Exception:
            pass
        self._ready.set()
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._ready = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._ready.wait(timeout=10)  # short timed regions: NVML init happens before them
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        smax = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(self.samples)}


def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------


# EvalMod of the sparse (weight-refresh) bootstraps: "double_angle" (degree-31
# cos + 3 squarings, ~22 key switches, one more level, max error 5.7e-4 at
# P16) or the reference's "sine" (degree 119, ~69 key switches, 3.1e-4)
SPARSE_EVALMOD = os.environ.get("SPARSE_EVALMOD", "double_angle")
# BENCH_WEAK=1: cfg4 with 512 rows per GPU (the minibatch grows with the GPU
# count; reported as weak scaling).  Default: the reference's 512-row
# minibatch sharded over the GPUs (strong scaling).
WEAK = os.environ.get("BENCH_WEAK") == "1"


def zeros_ct(params, keys, level, seed=4242):
    """Encryption of zeros with a fixed seed: every rank starts from the same
    limbs (the split refresh needs identical (w, u) on all ranks; train()
    broadcasts instead)."""
    from paper_2210_02574_b200 import ckks

    return ckks.encrypt(ckks.encode(params, np.zeros(params.slot_count), level), keys,
                        rng_seed=seed)


# The N = 2^16 preset of every workload but cfg1: "p16s", the 128-bit-secure
# bootstrappable preset the north star names (h = 192), or "p16",
# the reference-parity preset (h = 64, insecure-test-only).  BENCH_PRESET
# selects it; BENCH_BOOT_PRESET overrides it for cfg3.
PRESET = os.environ.get("BENCH_PRESET", "p16s")
BOOT_PRESET = os.environ.get("BENCH_BOOT_PRESET", PRESET)


def boot_preset():
    from paper_2210_02574_b200 import ckks

    return ckks.get_preset(BOOT_PRESET)


def p16():
    from paper_2210_02574_b200 import ckks

    return ckks.get_preset(PRESET)


class KsWorkload:
    """cfg2: 64 ciphertexts at the full P16 chain: NTT + iNTT of every limb and a
    relinearising key switch of every c1 (one batched launch sequence)."""

    metric = "key switches/sec"
    unit = "KS/s"
    higher = True
    batch = 64

    def setup(self, rank, world):
        import torch

        from paper_2210_02574_b200 import ckks, ring

        self.params = p16()
        self.keys = ckks.keygen(self.params, rotation_steps=[1], rng_seed=7,
                                include_conjugation=False)
        L = self.params.max_level
        n = self.params.ring_degree
        host = np.empty((self.batch, 2, L + 1, n), dtype=np.uint64)
        for i in range(self.batch):
            rng = np.random.default_rng(1000 + i + rank * self.batch)
            for c in range(2):
                for j, q in enumerate(self.params.ring.moduli_chain):
                    host[i, c, j] = rng.integers(0, q, size=n, dtype=np.uint64)
        self.host = torch.from_numpy(host.view(np.int64)).pin_memory()
        self.dev = self.host.to("cuda")
        self.out_host = torch.empty((self.batch, 2, L + 1, n), dtype=torch.int64).pin_memory()
        self.h2d = self.host.numel() * 8
        self.d2h = self.out_host.numel() * 8
        self.units = self.batch * world
        self.config = {"workload": "cfg2 NTT/iNTT + key-switch microbench", "preset": PRESET,
                       "N": n, "level": L, "ciphertexts_per_gpu": self.batch,
                       "l2": "inputs (1.4 GiB) exceed L2"}

    def _run(self, data):
        from paper_2210_02574_b200 import ring
        from paper_2210_02574_b200.ckks import keys as K

        params = self.params
        L = params.max_level
        sel = ring._dev.chain_primes(L + 1)
        ev = ring._dev.empty(*data.shape)
        ring._ntt_dev(params.ring, data, ev, L + 1, sel, False)  # all limbs -> eval
        back = ring._dev.empty(*data.shape)
        ring._ntt_dev(params.ring, ev, back, L + 1, sel, True)  # and back
        d = ring.RnsPoly(params.ring, ev[:, 1], ring.EVAL, L)
        kb, ka = K.ks_apply(self.keys, self.keys.relin_key, d)
        return kb, ka, back

    def step(self):
        return self._run(self.dev)

    def e2e_step(self):
        dev = self.host.to("cuda", non_blocking=True)
        kb, ka, _ = self._run(dev)
        self.out_host[:, 0].copy_(kb.data, non_blocking=True)
        self.out_host[:, 1].copy_(ka.data, non_blocking=True)

    def oracle_sample(self):
        """One KS at level L + NTT/iNTT of one ciphertext on the CPU oracle."""
        from oracle import scheme as S

        p = S.Params.from_text(self.params.to_config_text())
        if getattr(self, "_okeys", None) is None:
            self._okeys = S.keygen(p, [], 7, conj=False)
        keys = self._okeys
        rng = np.random.default_rng(1000)
        L = p.max_level
        d = np.stack([rng.integers(0, q, size=p.n, dtype=np.uint64) for q in p.chain])
        t0 = time.perf_counter()
        S.ntt_fwd(p, d, p.chain)
        S.ntt_fwd(p, d, p.chain)
        S.ntt_inv(p, d, p.chain)
        S.ntt_inv(p, d, p.chain)
        S.ks_apply(p, keys.relin, d, L)
        sec = time.perf_counter() - t0
        return 1.0 / sec, "1 ciphertext: 2x(22-limb NTT + iNTT) + 1 top-level KS (N=2^16)"


def cost_model_sample(params, histogram, units, unit_kind):
    """Reference CPU time of one step from the oracle cost model (bounded sample)."""
    from oracle.costmodel import OracleCostModel, histogram_levels

    t0 = time.perf_counter()
    model = OracleCostModel(params.to_config_text())
    ks_levels, other = histogram_levels(histogram)
    model.sample(ks_levels, other)
    sec = model.seconds(histogram)
    n_ks = sum(v for k, v in histogram.items() if k.startswith("ks@"))
    n_enc = sum(v for k, v in histogram.items() if k.startswith("encode@"))
    cal = reference_calibration(unit_kind, units)
    sample = (f"oracle (C/OpenMP, all host cores) timed KS at levels {ks_levels} and "
              f"encode/rescale/pt-mult at levels {other} ({time.perf_counter() - t0:.1f}s of "
              f"CPU sampling), weighted by the step's reference op histogram ({n_ks} KS, "
              f"{n_enc} encodes): modelled {sec:.1f} s per step")
    if cal is not None:
        sec *= cal["measured_over_model"]
        sample += (f"; x {cal['measured_over_model']:.3f} = the measured/modelled ratio of one "
                   f"full reference minibatch timed end to end ({cal['source']}): "
                   f"{sec:.1f} s per step")
    value = units / sec if unit_kind == "rate" else sec * 1e3
    return value, sample


_CONFIG = ["train"]  # the workload this process runs (set by main)


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def reference_calibration(unit_kind, units):
    """Measured/modelled ratio of the reference CPU path: one whole cfg4
    minibatch of the reference itself (numba, all cores) timed end to end
    next to this cost model on the same machine (tools/ref_minibatch_time.py,
    profiles/r02_ref_minibatch_time.log).  Applied to the train workload
    only, the one it was measured on."""
    if _CONFIG[0] != "train":
        return None
    path = os.path.join(REPO, "profiles", "r02_ref_minibatch_time.log")
    try:
        recs = [json.loads(ln) for ln in open(path) if ln.strip().startswith("{")]
        ref = next(r for r in recs if "minibatch_seconds" in r)
        mod = next(r for r in recs if "measured_over_model" in r)
    except (OSError, StopIteration, ValueError):
        return None
    return {"measured_over_model": float(mod["measured_over_model"]),
            "source": f"reference {ref['minibatch_seconds']:.0f} s vs model "
                      f"{mod['model_minibatch_seconds']:.0f} s on {ref['cores']} cores, "
                      "profiles/r02_ref_minibatch_time.log"}


def diag_gib(ctx):
    """HBM held by a context's diagonal cache (and its packed-pair context's)."""
    total = ctx.diag_cache_bytes()
    packed = getattr(ctx, "_packed_ctx", None)
    if packed is not None:
        total += packed.diag_cache_bytes()
    return total / 2 ** 30


def torch_stack_host(ct):
    """Device -> host read of a whole ciphertext (both components)."""
    import torch

    return torch.stack([ct.c0.data, ct.c1.data]).cpu()


class BootstrapWorkload:
    """cfg3: one sparse-1024 periodic bootstrap at N=2^16 (the w/u refresh)."""

    metric = "CKKS bootstrap ms (N=2^16)"
    unit = "ms"
    higher = False

    def setup(self, rank, world):
        import torch

        from paper_2210_02574_b200 import bootstrap as bs, ckks

        self.params = boot_preset()
        self.ctx = bs.build_context(self.params, n_slots=1024, input_periodic=True,
                                    evalmod=SPARSE_EVALMOD)
        steps = self.ctx.required_rotation_steps()
        t0 = time.time()
        self.keys = ckks.keygen(self.params, rotation_steps=steps, rng_seed=7)
        self.keygen_s = time.time() - t0
        v = np.tile(np.random.default_rng(1002).uniform(-1, 1, 1024), 32)
        self.v = v
        self.ct = ckks.encrypt_vector(self.params, v, self.keys, level=0, rng_seed=5)
        self.host = torch.stack([self.ct.c0.data, self.ct.c1.data]).cpu().pin_memory()
        self.h2d = self.host.numel() * 8
        self.d2h = 0
        self.units = 1
        self.config = {"workload": "cfg3 sparse-1024 periodic bootstrap", "preset": BOOT_PRESET,
                       "N": self.params.ring_degree, "n_slots": 1024,
                       "rotation_keys": len(steps)}

        self.captured = None
        if os.environ.get("BENCH_GRAPH", "1") == "1":
            # the bootstrap's ~5k launches replayed as one CUDA graph
            self.captured = bs.CapturedBootstrap(self.ct, self.ctx, self.keys)
            self.config["graph"] = "bootstrap captured as a CUDA graph"

    def step(self):
        from paper_2210_02574_b200 import bootstrap as bs

        if self.captured is not None:
            self.out = self.captured.run(self.ct)
        else:
            self.out = bs.bootstrap(self.ct, self.ctx, self.keys)
        return self.out

    def profile_step(self):
        from paper_2210_02574_b200 import bootstrap as bs

        return bs.bootstrap(self.ct, self.ctx, self.keys)

    def e2e_step(self):
        from paper_2210_02574_b200 import bootstrap as bs
        from paper_2210_02574_b200.ckks import ops

        if self.captured is not None:
            out = self.captured.run(self.host.to("cuda", non_blocking=True))
        else:
            t = ops._packed(self.params, (), 0)
            t.copy_(self.host.to("cuda", non_blocking=True))
            ct = ops._ct(t, 0, self.ct.scale, self.ct.slot_count, self.params)
            out = bs.bootstrap(ct, self.ctx, self.keys)
        self.d2h = out.c0.data.numel() * 16
        host = torch_stack_host(out)
        return host

    def oracle_sample(self):
        return cost_model_sample(self.params, self.histogram, 1, "ms")

    def check(self):
        from paper_2210_02574_b200 import ckks

        got = ckks.decrypt_vector(self.out, self.keys)
        return {"max_abs_err": float(np.max(np.abs(got - self.v))),
                "output_level": self.out.level, "keygen_s": round(self.keygen_s, 1),
                "diag_cache_gib": round(diag_gib(self.ctx), 2)}


class BootstrapFullWorkload:
    """cfg3 (full): full-slot bootstrap (32,768 slots) at N=2^16, B ciphertexts
    per step (BENCH_FULL_BATCH, default 1; B > 1 is the batched data-ingest
    refresh of logreg.py:338).  Its 196,609 diagonals are generated and encoded
    on the GPU every step (the reference encodes them on the host, ~2 h per
    bootstrap at N=2^16).  Metric: ms per refreshed ciphertext."""

    metric = "CKKS bootstrap ms (N=2^16)"
    unit = "ms"
    higher = False

    def setup(self, rank, world):
        import torch

        from paper_2210_02574_b200 import bootstrap as bs, ckks
        from paper_2210_02574_b200.ckks import ops

        self.params = boot_preset()
        slots = self.params.slot_count
        self.ctx = bs.build_context(self.params, n_slots=slots)
        steps = self.ctx.required_rotation_steps()
        t0 = time.time()
        self.keys = ckks.keygen(self.params, rotation_steps=steps, rng_seed=7)
        self.keygen_s = time.time() - t0
        self.batch = int(os.environ.get("BENCH_FULL_BATCH", "1"))
        self.ms_div = self.batch
        rng = np.random.default_rng(1002)
        self.vs = [rng.uniform(-1, 1, slots) for _ in range(self.batch)]
        self.cts = [ckks.encrypt_vector(self.params, v, self.keys, level=0, rng_seed=5 + i)
                    for i, v in enumerate(self.vs)]
        self.ct = self.cts[0] if self.batch == 1 else ops.stack(self.cts)
        self.host = torch.stack([self.ct.c0.data, self.ct.c1.data]).cpu().pin_memory()
        self.h2d = self.host.numel() * 8
        self.d2h = 0
        self.units = 1
        self.config = {"workload": "cfg3 full-slot bootstrap (32768 slots)", "preset": BOOT_PRESET,
                       "N": self.params.ring_degree, "n_slots": slots,
                       "ciphertexts_per_step": self.batch, "rotation_keys": len(steps),
                       "unit_note": "ms per refreshed ciphertext (step time / batch)",
                       "diagonals": "generated + encoded on the GPU every step"}

    def _boot(self, ct):
        from paper_2210_02574_b200 import bootstrap as bs
        from paper_2210_02574_b200.ckks import ops

        if ct.batch is None:
            return [bs.bootstrap(ct, self.ctx, self.keys)]
        return bs.bootstrap_many(ops.unstack(ct), self.ctx, self.keys)

    def step(self):
        self.outs = self._boot(self.ct)
        return self.outs

    def e2e_step(self):
        from paper_2210_02574_b200.ckks import ops

        lead = () if self.ct.batch is None else (self.ct.batch,)
        t = ops._packed(self.params, lead, 0)
        t.copy_(self.host.to("cuda", non_blocking=True).transpose(0, 1) if lead
                else self.host.to("cuda", non_blocking=True))
        ct = ops._ct(t, 0, self.ct.scale, self.ct.slot_count, self.params)
        outs = self._boot(ct)
        self.d2h = sum(o.c0.data.numel() * 16 for o in outs)
        return [torch_stack_host(o) for o in outs]

    def oracle_sample(self):
        return cost_model_sample(self.params, self.histogram, 1, "ms")

    def check(self):
        from paper_2210_02574_b200 import ckks

        errs = [float(np.max(np.abs(ckks.decrypt_vector(o, self.keys) - v)))
                for o, v in zip(self.outs, self.vs)]
        err = max(errs)
        # north star: <= 1e-3; the reference preset's documented bound 2.5e-3
        # (EvalMod noise at scale 2^40) -- gated, not only reported
        bound = 1e-3 if BOOT_PRESET == "p16s" else 2.5e-3
        if err > bound:
            raise SystemExit(f"full-slot bootstrap error {err:.3e} exceeds {bound:.1e}")
        return {"max_abs_err": err, "within_1e-3": err <= 1e-3, "error_bound_checked": bound,
                "output_level": self.outs[0].level, "keygen_s": round(self.keygen_s, 1)}


class PredictWorkload:
    """cfg1: N=2^14 (P14) encrypted 768-d logistic-regression inference on one
    ciphertext of 8 rows: step = encrypt the rows ->
    predict (encrypted dot product + degree-15 sigmoid) -> decrypt the scores.
    Metric: ms per inference (latency; the reference: 0.106 / 2.64 / 0.004 s)."""

    metric = "encrypted LR inference ms (N=2^14, 8 rows)"
    unit = "ms"
    higher = False

    def setup(self, rank, world):
        from paper_2210_02574_b200 import ckks, logreg, minimax

        self.params = ckks.get_preset("p14")
        t0 = time.time()
        self.keys = ckks.keygen(self.params, rng_seed=7)
        self.keygen_s = time.time() - t0
        self.layout = logreg.make_layout(self.params, 768)
        self.sig = minimax.load_approximant("sigmoid_deg15")
        self.X = np.random.default_rng(0).uniform(-1, 1, (8, 768))
        w = np.random.default_rng(0).normal(0, 0.05, 768)
        wv = np.zeros(self.layout.slot_count)
        for b in range(self.layout.rows_per_ct):
            wv[b * self.layout.padded_dim: b * self.layout.padded_dim + 768] = w
        wct = ckks.encrypt_vector(self.params, wv, self.keys, rng_seed=2)
        self.model = logreg.EncryptedModel(2, self.layout, [wct], [wct])
        self.wpad = np.concatenate([w, np.zeros(self.layout.padded_dim - 768)])[None, :]
        self.slots = logreg._pack_slots(self.X, self.layout)
        self.units = 1
        self.h2d = self.layout.slot_count * 8  # the packed rows (encoded and encrypted on device)
        self.d2h = 0
        self.config = {"workload": "cfg1 P14 encrypt -> 768-d LR inference -> decrypt, 1 ct",
                       "preset": "p14", "N": self.params.ring_degree, "rows": 8}

    def step(self):
        from paper_2210_02574_b200 import ckks, logreg

        ct = ckks.encrypt_vector(self.params, self.slots, self.keys, rng_seed=1)
        self.scores = logreg.predict(self.model, [ct], self.keys, self.sig)
        self.dec = logreg.decrypt_scores(self.scores, self.keys, self.layout, 8)
        self.d2h = 2 * (self.scores[0][0].level + 1) * self.params.ring_degree * 8
        return self.dec

    e2e_step = step  # host rows in, host scores out: the step is already end to end

    def oracle_sample(self):
        return cost_model_sample(self.params, self.histogram, 1, "ms")

    def check(self):
        from paper_2210_02574_b200 import logreg

        want = logreg.shadow_scores(self.X, self.wpad, self.sig, self.layout)
        return {"max_abs_err_vs_shadow": float(np.max(np.abs(self.dec - want))),
                "keygen_s": round(self.keygen_s, 1)}


def logreg_rotation_steps(layout):
    """Rotation steps of the gradient pipeline (logreg.py:202-229): the
    reference's doubling steps plus the multiples the hoisted radix-4 rounds
    use (logreg.rotation_steps)."""
    from paper_2210_02574_b200 import logreg

    return logreg.rotation_steps(layout)


class TrainWorkload:
    """cfg4 (SST-2-sized synthetic 768-d embeddings, P16): one minibatch of the
    encrypted Nesterov trainer = 16 ciphertexts x 32 rows (batch 512), the
    batched gradient, the modular gradient sum, the update and the
    sparse-1024 bootstrap refresh of w and u.  Data ciphertexts are at the
    refresher's output level (the reference excludes the ingest refresh from
    epoch time, logreg.py:337-339)."""

    metric = "encrypted LR train samples/sec"
    unit = "samples/s"
    higher = True
    batch_rows = 512
    n_pool = 4  # distinct minibatches cycled through

    def setup(self, rank, world):
        import torch

        from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg, minimax, shard
        from paper_2210_02574_b200.ckks import ops
        from paper_2210_02574_b200.synth import make_separable

        if WEAK and type(self) is TrainWorkload:  # 512 rows per GPU: the minibatch grows with N
            self.batch_rows = TrainWorkload.batch_rows * world

        self.params = params = p16()
        self.sig = minimax.load_approximant("sigmoid_deg15")
        self.layout = logreg.make_layout(params, 768)
        self.ctx = bs.build_context(params, n_slots=self.layout.padded_dim, input_periodic=True,
                                    evalmod=SPARSE_EVALMOD)
        steps = sorted(set(bs.refresh_rotation_steps(self.ctx)) | logreg_rotation_steps(self.layout))
        t0 = time.time()
        self.keys = ckks.keygen(params, rotation_steps=steps, rng_seed=7)
        self.keygen_s = time.time() - t0
        self.refresher = bs.BootstrapRefresher(self.ctx, self.keys)
        self.cfg = logreg.TrainConfig(1.0, 0.9, self.batch_rows, 1)
        rows_per_ct = self.layout.rows_per_ct
        cts = self.batch_rows // rows_per_ct
        lo, hi = shard.shard_range(cts, rank, world)
        self.local = hi - lo
        X, y = make_separable(np.random.default_rng(100), self.batch_rows * self.n_pool, dim=768,
                              margin=0.5)
        self.X, self.y = X, y
        top = self.ctx.output_level
        self.pool_dev = []
        for b in range(self.n_pool):
            xs, ys = [], []
            for c in range(lo, hi):
                r0 = b * self.batch_rows + c * rows_per_ct
                xr, yr = X[r0 : r0 + rows_per_ct], y[r0 : r0 + rows_per_ct]
                xs.append(ckks.encrypt(ckks.encode(params, logreg._pack_slots(xr, self.layout), top),
                                       self.keys, rng_seed=10_000 + b * 100 + c))
                ys.append(ckks.encrypt(
                    ckks.encode(params, logreg._pack_label_slots(yr, self.layout), 3), self.keys,
                    rng_seed=20_000 + b * 100 + c))
            self.pool_dev.append((ops.stack(xs), ops.stack(ys)))
        # pinned host copies of each minibatch's ciphertexts (the e2e leg uploads them)
        self.host_x = [torch.stack([xb.c0.data, xb.c1.data], dim=1).cpu().pin_memory()
                       for xb, _ in self.pool_dev]
        self.host_y = [torch.stack([yb.c0.data, yb.c1.data], dim=1).cpu().pin_memory()
                       for _, yb in self.pool_dev]
        self.w = zeros_ct(params, self.keys, top)
        self.u = zeros_ct(params, self.keys, top)
        self.it = 0
        self.graph = self.sgraph = None
        if os.environ.get("BENCH_GRAPH", "1") == "1":
            xb, yb = self.pool_dev[0]
            if world == 1 and os.environ.get("BENCH_SHARDED_GRAPH") != "1":
                self.graph = logreg.CapturedMinibatch(self.w, self.u, xb, yb, self.batch_rows,
                                                      self.cfg, self.keys, self.sig, self.layout,
                                                      self.refresher)
            else:  # per-rank gradient graph + owner refresh graphs, eager collectives
                self.sgraph = logreg.CapturedShardedMinibatch(
                    self.w, self.u, xb, yb, self.batch_rows, self.cfg, self.keys, self.sig,
                    self.layout, self.refresher)
            # (the capture warm-up updated a throwaway copy; the state is still the initial one)
        self.units = self.batch_rows
        self.h2d = (self.host_x[0].numel() + self.host_y[0].numel()) * 8
        self.d2h = 0
        self.config = self.static_config(world)
        self.config["rotation_keys"] = len(steps)
        if self.graph is not None:
            self.config["e2e_pipeline"] = ("minibatch i+1 copied H2D from pinned host memory on a "
                                           "side stream during step i; w copied D2H every step")

    @classmethod
    def static_config(cls, world):
        return {
            "workload": "cfg4 encrypted-LR training minibatch (SST-2-shaped synthetic 768-d)",
            "preset": PRESET, "N": 65536,
            "batch_rows": cls.batch_rows * (world if WEAK else 1),
            "ciphertexts_per_minibatch": cls.batch_rows * (world if WEAK else 1) // 32,
            "rows_per_ct": 32,
            "refresh": "w and u refreshed together: one packed sparse bootstrap of period 2048 (two of period 1024 in the reference)",
            "evalmod": SPARSE_EVALMOD,
            "parallelism": f"minibatch sharded over {world} GPU(s)",
            "l2": "inputs exceed L2 (126 MB): keys ~30 GiB, run-compressed diagonals ~10 GiB, minibatch 0.3 GiB"}

    def profile_step(self):
        """Eager (un-captured) step: per-launch profile and op histogram."""
        from paper_2210_02574_b200 import logreg

        xb, yb = self.pool_dev[self.it % self.n_pool]
        self.it += 1
        w, u = logreg.train_minibatch(
            self.w, self.u, xb, yb, self.batch_rows, self.cfg, self.keys, self.sig, self.layout,
            self.refresher, local_shard=True)
        if self.graph is not None:  # keep the captured state in sync
            for dst, src in ((self.graph.w, w), (self.graph.u, u)):
                dst.c0.data.copy_(src.c0.data)
                dst.c1.data.copy_(src.c1.data)
            self.w, self.u = self.graph.w, self.graph.u
        else:
            self.w, self.u = w, u

    def step(self):
        from paper_2210_02574_b200 import logreg

        xb, yb = self.pool_dev[self.it % self.n_pool]
        self.it += 1
        if self.graph is not None:
            self.graph.load(xb, yb)
            self.w, self.u = self.graph.step()
            return self.w
        if self.sgraph is not None:
            self.sgraph.load(xb, yb)
            self.w, self.u = self.sgraph.step()
            return self.w
        self.w, self.u = logreg.train_minibatch(
            self.w, self.u, xb, yb, self.batch_rows, self.cfg, self.keys, self.sig, self.layout,
            self.refresher, local_shard=True)
        return self.w

    def e2e_step(self):
        from paper_2210_02574_b200 import logreg
        from paper_2210_02574_b200.ckks import ops

        i = self.it % self.n_pool
        self.it += 1
        if self.graph is not None:
            # pipelined input: this step's minibatch was copied H2D (pinned host
            # memory) during the previous step; the next one's copy starts now
            # and overlaps this replay.  Every step does one H2D and one D2H.
            if not getattr(self, "_prefetched", False):
                self.graph.prefetch(self.host_x[i], self.host_y[i])
                self._prefetched = True
            self.graph.load_prefetched()
            nxt = self.it % self.n_pool
            self.graph.prefetch(self.host_x[nxt], self.host_y[nxt])
            self.w, self.u = self.graph.step()
            if getattr(self, "_w_host", None) is None:
                import torch

                self._w_host = torch.empty((2,) + tuple(self.w.c0.data.shape),
                                           dtype=self.w.c0.data.dtype, pin_memory=True)
            self._w_host[0].copy_(self.w.c0.data, non_blocking=True)  # D2H of the result
            self._w_host[1].copy_(self.w.c1.data, non_blocking=True)
            self.d2h = self._w_host.numel() * 8
            return self._w_host
        if self.sgraph is not None:
            self.sgraph.load(self.host_x[i], self.host_y[i])  # H2D from pinned host memory
            self.w, self.u = self.sgraph.step()
            wh = self.w.c0.data.to("cpu")
            wh1 = self.w.c1.data.to("cpu")
            self.d2h = (wh.numel() + wh1.numel()) * 8
            return wh, wh1
        xt = self.host_x[i].to("cuda", non_blocking=True)
        yt = self.host_y[i].to("cuda", non_blocking=True)
        x0, y0 = self.pool_dev[i]
        xb = ops._ct(xt, x0.level, x0.scale, x0.slot_count, self.params)
        yb = ops._ct(yt, y0.level, y0.scale, y0.slot_count, self.params)
        self.w, self.u = logreg.train_minibatch(
            self.w, self.u, xb, yb, self.batch_rows, self.cfg, self.keys, self.sig, self.layout,
            self.refresher, local_shard=True)
        wh = self.w.c0.data.to("cpu", non_blocking=False)
        self.d2h = wh.numel() * 8 * 2
        wh1 = self.w.c1.data.to("cpu")
        return wh, wh1

    def oracle_sample(self):
        return cost_model_sample(self.params, self.histogram, self.units, "rate")

    def check(self):
        """Validation run: from w = u = 0, apply the first two minibatches
        (the reference acceptance test's protocol, T/test_acceptance.py:98-131)
        and compare the decrypted weights with the plaintext shadow trainer."""
        from paper_2210_02574_b200 import ckks, logreg

        top = self.ctx.output_level
        zero_w = zeros_ct(self.params, self.keys, top)
        zero_u = zeros_ct(self.params, self.keys, top)
        g = self.graph if self.graph is not None else self.sgraph
        if g is not None:
            for dst, src in ((g.w, zero_w), (g.u, zero_u)):
                dst.c0.data.copy_(src.c0.data)
                dst.c1.data.copy_(src.c1.data)
            self.w, self.u = g.w, g.u
        else:
            self.w, self.u = zero_w, zero_u
        self.it = 0
        n_check = 2
        for _ in range(n_check):
            self.step()
        w = ckks.decrypt_vector(self.w, self.keys)[: self.layout.padded_dim]
        Xs = self.X[: n_check * self.batch_rows]
        ys = self.y[: n_check * self.batch_rows]
        sh = logreg.shadow_train(Xs, ys, self.cfg, self.sig, layout=self.layout)
        return {"weights_vs_shadow_max_abs": float(np.max(np.abs(w - sh.weights[0]))),
                "validation_minibatches": n_check, "keygen_s": round(self.keygen_s, 1),
                "diag_cache_gib": round(diag_gib(self.ctx), 2)}


class OvrWorkload(TrainWorkload):
    """cfg5 (AG-News-sized synthetic 1024-d embeddings, 4 classes, P16): one
    minibatch of One-vs-Rest training (the reference's multi-class semantics,
    logreg.py:325-331, 393-398) = the same 32 data ciphertexts x 16 rows
    (batch 512) against the 4 classes' label ciphertexts, each class's
    Nesterov update and its sparse-2048 bootstrap refresh of w and u (one
    batch of two).
    A step updates all 4 class-models; samples/s counts rows (each row
    updates every class).  Classes are independent (no exchange): under
    torchrun the classes are dealt round-robin to the ranks (N <= 4)."""

    metric = "encrypted OvR train samples/sec (4 class-models)"
    n_pool = 2
    n_classes = 4
    dim = 1024

    def setup(self, rank, world):
        import torch

        from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg, minimax
        from paper_2210_02574_b200.ckks import ops
        from paper_2210_02574_b200.synth import make_blob_embeddings

        from paper_2210_02574_b200 import shard

        # 2-D layout (shard.class_groups): world <= 4 deals the classes to
        # ranks; world = 4k gives each class k ranks sharding its minibatch
        members = shard.class_groups(self.n_classes, world)
        self.cgroup = {}
        if world > 1:
            import torch.distributed as dist

            made = {}
            for c, m in enumerate(members):
                key = tuple(m)
                if key not in made:
                    made[key] = None if len(m) == world else dist.new_group(list(m))
                self.cgroup[c] = made[key]
        self.members = members
        self.params = params = p16()
        self.sig = minimax.load_approximant("sigmoid_deg15")
        self.layout = logreg.make_layout(params, self.dim)
        self.ctx = bs.build_context(params, n_slots=self.layout.padded_dim, input_periodic=True,
                                    evalmod=SPARSE_EVALMOD)
        steps = sorted(set(bs.refresh_rotation_steps(self.ctx)) | logreg_rotation_steps(self.layout))
        t0 = time.time()
        self.keys = ckks.keygen(params, rotation_steps=steps, rng_seed=7)
        self.keygen_s = time.time() - t0
        self.refresher = bs.BootstrapRefresher(self.ctx, self.keys)
        self.cfg = logreg.TrainConfig(0.5, 0.9, self.batch_rows, 1)  # T/test_acceptance.py:151-154
        self.mine = [c for c in range(self.n_classes) if rank in members[c]]
        rpc = self.layout.rows_per_ct
        n_cts = self.batch_rows // rpc
        m0 = members[self.mine[0]]
        ct_lo, ct_hi = shard.shard_range(n_cts, m0.index(rank), len(m0))  # this rank's cts
        n_per_class = self.batch_rows * self.n_pool // self.n_classes
        X, y = make_blob_embeddings(np.random.default_rng(200), n_per_class, self.n_classes,
                                    dim=self.dim)
        self.X, self.y = X, y
        top = self.ctx.output_level
        self.pool_dev = []
        for b in range(self.n_pool):
            xs, ys = [], {c: [] for c in self.mine}
            for i in range(ct_lo, ct_hi):
                r0 = b * self.batch_rows + i * rpc
                xs.append(ckks.encrypt(
                    ckks.encode(params, logreg._pack_slots(X[r0 : r0 + rpc], self.layout), top),
                    self.keys, rng_seed=30_000 + b * 1000 + i))
                for c in self.mine:
                    yc = (y[r0 : r0 + rpc] == c).astype(np.float64)
                    ys[c].append(ckks.encrypt(
                        ckks.encode(params, logreg._pack_label_slots(yc, self.layout), 3),
                        self.keys, rng_seed=40_000 + b * 1000 + c * 100 + i))
            self.pool_dev.append((ops.stack(xs), {c: ops.stack(ys[c]) for c in self.mine}))
        self.host_x = [torch.stack([xb.c0.data, xb.c1.data], dim=1).cpu().pin_memory()
                       for xb, _ in self.pool_dev]
        self.host_y = [{c: torch.stack([yb[c].c0.data, yb[c].c1.data], dim=1).cpu().pin_memory()
                        for c in self.mine} for _, yb in self.pool_dev]
        self.w = {c: zeros_ct(params, self.keys, top) for c in self.mine}
        self.u = {c: zeros_ct(params, self.keys, top) for c in self.mine}
        self.it = 0
        xb, yb = self.pool_dev[0]
        # one captured minibatch per class (independent state, same data shape)
        # (replayed in capture order every step, so they share one graph pool)
        self.graphs, pool = {}, None
        for c in self.mine:
            if len(members[c]) > 1:  # this class's minibatch sharded over its group
                self.w[c] = shard.broadcast_ciphertext(self.w[c], 0, self.w[c], self.cgroup[c])
                self.u[c] = shard.broadcast_ciphertext(self.u[c], 0, self.u[c], self.cgroup[c])
                self.graphs[c] = logreg.CapturedShardedMinibatch(
                    self.w[c], self.u[c], xb, yb[c], self.batch_rows, self.cfg, self.keys,
                    self.sig, self.layout, self.refresher, group=self.cgroup[c])
                continue
            g = logreg.CapturedMinibatch(self.w[c], self.u[c], xb, yb[c], self.batch_rows,
                                         self.cfg, self.keys, self.sig, self.layout,
                                         self.refresher, pool=pool)
            self.graphs[c], pool = g, g.pool
        self.graph = self.sgraph = None
        import types

        self.captured = types.SimpleNamespace(
            kernels_per_run=sum(g.kernels_per_step for g in self.graphs.values()))
        self.units = self.batch_rows
        self.h2d = (self.host_x[0].numel() + sum(t.numel() for t in self.host_y[0].values())) * 8
        self.d2h = 0
        self.config = self.static_config(world)
        self.config["rotation_keys"] = len(steps)
        self.config["classes_on_this_rank"] = self.mine

    @classmethod
    def static_config(cls, world):
        return {
            "workload": "cfg5 encrypted One-vs-Rest training minibatch (AG-News-shaped "
                        "synthetic 1024-d, 4 classes)",
            "preset": PRESET, "N": 65536, "batch_rows": cls.batch_rows,
            "classes": cls.n_classes, "ciphertexts_per_minibatch": cls.batch_rows // 16,
            "rows_per_ct": 16,
            "refresh": "per class: w and u refreshed as one batch of two sparse-2048 "
                       "bootstraps (pair packing stops at period 1024: bootstrap.PACKED_PAIR_MAX_SLOTS)",
            "parallelism": (f"classes dealt round-robin over {world} GPU(s), no exchange"
                            if world <= cls.n_classes else
                            f"2-D: {cls.n_classes} class groups x {world // cls.n_classes} ranks "
                            "sharding each class's minibatch (split refresh)"),
            "l2": "keys and diagonals exceed L2"}

    def profile_step(self):
        from paper_2210_02574_b200 import logreg

        import torch

        torch.cuda.empty_cache()  # the eager step allocates outside the graph pool
        xb, yb = self.pool_dev[self.it % self.n_pool]
        self.it += 1
        for c, g in self.graphs.items():
            grp = self.cgroup.get(c) if len(self.members[c]) > 1 else logreg._SOLO
            w, u = logreg.train_minibatch(g.w, g.u, xb, yb[c], self.batch_rows, self.cfg,
                                          self.keys, self.sig, self.layout, self.refresher,
                                          local_shard=True, group=grp)
            for dst, src in ((g.w, w), (g.u, u)):
                dst.c0.data.copy_(src.c0.data)
                dst.c1.data.copy_(src.c1.data)

    def step(self):
        xb, yb = self.pool_dev[self.it % self.n_pool]
        self.it += 1
        for c, g in self.graphs.items():
            g.load(xb, yb[c])
            self.w[c], self.u[c] = g.step()
        return self.w

    def e2e_step(self):
        """Public-API step from pinned host buffers: the data ciphertexts are
        copied H2D once (into the first class's graph, then device-to-device
        into the others), each class's labels once; every class's refreshed w
        is read back."""
        import torch

        i = self.it % self.n_pool
        self.it += 1
        first = None
        for c, g in self.graphs.items():
            if first is None:
                g.load(self.host_x[i], self.host_y[i][c])
                first = g
            else:
                g.load(first.x, self.host_y[i][c])
            self.w[c], self.u[c] = g.step()
        if getattr(self, "_w_host", None) is None:
            w0 = next(iter(self.w.values()))
            self._w_host = torch.empty((len(self.w), 2) + tuple(w0.c0.data.shape),
                                       dtype=w0.c0.data.dtype, pin_memory=True)
        for k, c in enumerate(self.mine):
            self._w_host[k, 0].copy_(self.w[c].c0.data, non_blocking=True)
            self._w_host[k, 1].copy_(self.w[c].c1.data, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        self.d2h = self._w_host.numel() * 8
        return self._w_host

    def check(self):
        """From w = u = 0 every class applies the first minibatch; decrypted
        weights against the plaintext OvR shadow trainer (T/test_acceptance.py:
        151-171 protocol)."""
        from paper_2210_02574_b200 import ckks, logreg

        top = self.ctx.output_level
        for g in self.graphs.values():
            for dst in (g.w, g.u):
                z = zeros_ct(self.params, self.keys, top)
                dst.c0.data.copy_(z.c0.data)
                dst.c1.data.copy_(z.c1.data)
        self.it = 0
        self.step()
        sh = logreg.shadow_train(self.X[: self.batch_rows], self.y[: self.batch_rows], self.cfg,
                                 self.sig, class_count=self.n_classes, layout=self.layout)
        err = 0.0
        for c in self.mine:
            w = ckks.decrypt_vector(self.w[c], self.keys)[: self.layout.padded_dim]
            err = max(err, float(np.max(np.abs(w - sh.weights[c]))))
        return {"weights_vs_shadow_max_abs": err, "validation_minibatches": 1,
                "keygen_s": round(self.keygen_s, 1),
                "diag_cache_gib": round(diag_gib(self.ctx), 2)}


WORKLOADS = {"train": TrainWorkload, "ks": KsWorkload, "bootstrap": BootstrapWorkload,
             "bootstrap_full": BootstrapFullWorkload, "predict": PredictWorkload,
             "ovr": OvrWorkload}


# ---------------------------------------------------------------------------
# timing
# ---------------------------------------------------------------------------


def timed(fn, steps, world):
    import torch

    barrier(world)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        fn()
    b.record(stream)
    b.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    return a.elapsed_time(b)


def run_ours(args):
    import torch

    from paper_2210_02574_b200 import _lib

    rank, world = init_dist(args)
    wl = WORKLOADS[args.config]()
    wl.setup(rank, world)
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()
    n0 = _lib.launch_count()
    with ClockSampler(0 if os.environ.get("BENCH_ONE_DEVICE_GLOO") == "1" else int(os.environ.get("LOCAL_RANK", 0))) as clk:
        ms = timed(wl.step, args.steps, world)
    launches = _lib.launch_count() - n0
    graph = getattr(wl, "graph", None)
    if graph is not None:  # kernels replayed from the captured graph
        launches += graph.kernels_per_step * args.steps
    captured = getattr(wl, "captured", None)
    if captured is not None:
        launches += captured.kernels_per_run * args.steps
    sgraph = getattr(wl, "sgraph", None)
    if sgraph is not None:  # graph-replayed kernels (the eager ones are counted above)
        launches += sgraph.kernels_per_step * args.steps
    ms = max_over_ranks(ms, world)
    ms_step = ms / args.steps
    # end to end through the public API with host buffers
    wl.e2e_step()
    e2e_ms = max_over_ranks(timed(wl.e2e_step, max(1, args.steps // 2), world), world) / max(
        1, args.steps // 2)
    # per-kernel-class profile + reference op histogram of one step (separate
    # pass, not the timed one)
    from paper_2210_02574_b200 import _stats

    prof_step = wl.profile_step if hasattr(wl, "profile_step") else wl.step
    _lib.profile_enable(True)
    if os.environ.get("BENCH_NVTX"):  # lets ncu --nvtx-include "profile_step/" target one step
        torch.cuda.nvtx.range_push("profile_step")
    prof_step()
    if os.environ.get("BENCH_NVTX"):
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    # the reference op histogram in a separate pass: recording it may run the
    # reference's op sequence next to ours (e.g. the packed pair refresh)
    _stats.enable(True)
    prof_step()
    torch.cuda.synchronize()
    wl.histogram = _stats.snapshot()
    _stats.enable(False)
    div = getattr(wl, "ms_div", 1)
    if div > 1:  # per-unit histogram (the metric is time per ciphertext)
        wl.histogram = {k: v // div for k, v in wl.histogram.items()}
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    if rank == 0 and wl.histogram:
        with open(os.path.join(REPO, "gpurun_out", f"op_histogram_{args.config}.json"), "w") as fh:
            json.dump(wl.histogram, fh, indent=1, sort_keys=True)
    extra = wl.check() if hasattr(wl, "check") else {}
    if rank != 0:
        return
    if wl.higher:
        value = wl.units / (ms_step / 1e3)
        e2e_value = wl.units / (e2e_ms / 1e3)
    else:  # time per unit (a full-slot step refreshes `ms_div` ciphertexts)
        value = ms_step / getattr(wl, "ms_div", 1)
        e2e_value = e2e_ms / getattr(wl, "ms_div", 1)
    peak, peak_kind = measured_peaks()
    dom = max(prof, key=lambda c: prof[c]["ms"])
    dp = prof[dom]
    achieved = dp["bytes"] / (dp["ms"] / 1e3) / 1e9 if dp["ms"] else 0.0
    # ntt_modup / ntt_moddown / ntt_rescale are subsets of "ntt"
    step_ms_prof = sum(p["ms"] for c, p in prof.items() if not c.startswith("ntt_"))
    try:
        int_peak = _lib.modmul_peak()
        fp_peak = _lib.fp_modmul_peak()
    except Exception:
        int_peak = fp_peak = None
    mm_rate = dp["modmuls"] / (dp["ms"] / 1e3) if dp["ms"] else 0
    traffic, traffic_src = dram_traffic(args.config, dom)
    line = {
        "metric": wl.metric, "value": round(value, 4), "unit": wl.unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": wl.higher,
        "scaling": "weak" if (args.config == "ks" or (WEAK and args.config == "train")) else "strong",
        "vs_baseline": None, "dtype": "u64 (RNS residues mod 40-60-bit primes)",
        "data": "synthetic", "config": wl.config,
        "e2e": {"value": round(e2e_value, 4), "unit": wl.unit,
                "h2d_bytes_per_step": int(wl.h2d), "d2h_bytes_per_step": int(wl.d2h)},
        "gpu_launches": int(launches) if launches else None,
        "roofline": roofline_block(dom, dp, achieved, peak, peak_kind, mm_rate, int_peak,
                                   fp_peak, wl, traffic, traffic_src, step_ms_prof),
        # the NTT is modmul-bound, not HBM-bound: its products run on the FP64
        # pipe for primes < 2^46 and on the integer pipe (64-bit Shoup) for the
        # 60-bit primes; both peaks are measured by the library on this GPU
        "int_roofline": {
            "kernel": dom,
            "achieved_modmul_per_s": round(mm_rate, 1),
            "peak_modmul_per_s": int_peak,
            "frac": round(mm_rate / int_peak, 4) if (mm_rate and int_peak) else None,
            "fp64_peak_modmul_per_s": fp_peak,
            "frac_of_fp64_peak": round(mm_rate / fp_peak, 4) if (mm_rate and fp_peak) else None},
        "kernel_profile_ms": {c: round(p["ms"], 3) for c, p in prof.items() if p["launches"]},
        "kernel_profile_gbs": {c: round(p["bytes"] / p["ms"] / 1e6, 1)
                               for c, p in prof.items() if p["launches"] and p["ms"]},
        "kernel_profile_launches": {c: p["launches"] for c, p in prof.items() if p["launches"]},
        "clocks": clk.summary(),
    }
    line.update(extra)
    if hasattr(wl, "static_config"):  # the reference arm prints exactly this config
        static = wl.static_config(world)
        line["run_info"] = {k: v for k, v in wl.config.items() if k not in static}
        line["config"] = static
    line["cpu_baseline"] = cpu_baseline(wl)
    print(json.dumps(line), flush=True)


def roofline_block(dom, dp, achieved, peak, peak_kind, mm_rate, int_peak, fp_peak, wl, traffic,
                   traffic_src, step_ms_prof):
    """Roofline of the dominant kernel class against the bound it actually
    sits closer to: HBM bytes/s, or modular products/s against the blended
    modmul peak (FP64 products for primes < 2^46, 64-bit integer Shoup
    products for the rest, weighted by the preset's share of each)."""
    hbm_frac = achieved / peak if peak else 0.0
    blended = None
    if int_peak and fp_peak:
        primes = list(wl.params.ring.moduli_chain) + list(wl.params.ring.special_moduli)
        f = sum(1 for q in primes if q < (1 << 46)) / len(primes)
        blended = 1.0 / (f / fp_peak + (1.0 - f) / int_peak)
    mm_frac = mm_rate / blended if blended else 0.0
    base = {"kernel": dom, "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_bytes_per_launch": round(dp["bytes"] / dp["launches"])
            if dp["launches"] else None,
            "share_of_step": round(dp["ms"] / step_ms_prof, 4) if step_ms_prof else None,
            "hbm": {"achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                    "unit": "GB/s", "frac": round(hbm_frac, 4)},
            "modmul": {"achieved": round(mm_rate / 1e12, 4),
                       "peak": round(blended / 1e12, 4) if blended else None,
                       "unit": "Tmodmul/s", "frac": round(mm_frac, 4),
                       "peak_note": "blended FP64/INT64 modmul peak measured by the library"}}
    if mm_frac > hbm_frac:
        base.update({"bound": "int", "achieved": base["modmul"]["achieved"],
                     "peak": base["modmul"]["peak"], "unit": "Tmodmul/s",
                     "frac": round(mm_frac, 4)})
    else:
        base.update({"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(hbm_frac, 4)})
    return base


def dram_traffic(config, cls):
    """Measured DRAM bytes per launch of kernel class `cls` in this workload's
    step: profiles/<round>_dram_traffic_<config>.json, written by
    tools/dram_summary.py from an ncu pass (dram__bytes_read/write.sum) over
    one eager step of the same command (tools/profile_round.sh)."""
    import glob

    paths = sorted(glob.glob(os.path.join(REPO, "profiles", f"r*_dram_traffic_{config}.json")))
    if not paths:
        return None, None
    try:
        with open(paths[-1]) as fh:
            rec = json.load(fh)[cls]
        return int(rec["dram_bytes_per_launch"]), os.path.relpath(paths[-1], REPO)
    except (KeyError, ValueError, OSError):
        return None, None


def cpu_baseline(wl):
    try:
        from oracle import kernels as OK

        if OK.clib() is None:
            OK.build_c()
            OK._clib = None
        value, sample = wl.oracle_sample()
        return {"value": round(value, 6), "unit": wl.unit, "cores": os.cpu_count(),
                "kind": "port", "method": "oracle cost model (bounded sample)",
                "cpu": cpu_model(), "sample": sample}
    except Exception as exc:  # the baseline must never break the GPU line
        return {"value": None, "unit": wl.unit, "cores": os.cpu_count(), "kind": "port",
                "sample": f"unavailable: {exc}"}


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    wl = WORKLOADS[args.config]()

    from oracle.costmodel import load_histogram

    class _Preset:  # the preset file text only: nothing of the engine runs on this arm
        def __init__(self, path):
            with open(path) as fh:
                self.text = fh.read()

        def to_config_text(self):
            return self.text

    preset = "p14" if args.config == "predict" else (
        BOOT_PRESET if args.config.startswith("bootstrap") else PRESET)
    wl.params = _Preset(os.path.join(REPO, "paper_2210_02574_b200", "presets", f"{preset}.preset"))
    if args.config in ("train", "bootstrap", "bootstrap_full", "predict", "ovr"):
        try:  # the histogram recorded on this preset, else the P16 one
            wl.histogram = load_histogram(f"{args.config}_{preset}")
        except OSError:
            wl.histogram = load_histogram(args.config)
        # the modelled minibatch is the reference's 512 rows (samples/s does not
        # depend on how many minibatches a step holds)
        wl.units = TrainWorkload.batch_rows if args.config in ("train", "ovr") else 1
    vals = []
    for i in range(args.warmup + args.steps):
        v, sample = wl.oracle_sample()
        if i >= args.warmup:
            vals.append(v)
    value = float(np.median(vals))
    line = {"metric": wl.metric, "value": round(value, 6), "unit": wl.unit,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": wl.higher, "impl": "reference", "data": "synthetic",
            "config": (wl.static_config(args.gpus) if hasattr(wl, "static_config")
                       else {"workload": args.config, "preset": preset}),
            "cpu_baseline": {"value": round(value, 6), "unit": wl.unit,
                             "cores": os.cpu_count(), "kind": "port",
                             "method": "oracle cost model (bounded sample)", "cpu": cpu_model(),
                             "sample": sample},
            "e2e": {"value": round(value, 6), "unit": wl.unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    _CONFIG[0] = args.config
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
