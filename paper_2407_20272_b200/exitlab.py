"""Python mirror of the reference's engine / exit-policy API over the C ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/exitlab):

* ``ModelConfig``, ``ThresholdSchedule``, ``CostModel``, ``EngineConfig``  (model.hpp:18-25,
  exit_policy.hpp:36-42, engine.hpp:18-42)
* ``ExitTechnique.softmax_response() / state_similarity() / classifier() / never() /
  always_at(k)`` and ``technique_from_name`` (exit_policy.hpp:14-31)
* ``Engine(config).run(workload) -> Transcript``  (engine.hpp:131-147)
* errors: ``ValueError`` = std::invalid_argument, ``KvOutOfMemory`` (a RuntimeError) =
  exitlab::KvOutOfMemory, ``RuntimeError`` = std::runtime_error, ``LogicError`` = std::logic_error

Every compute call goes to libexitlab_b200.so on the GPU; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from .build import LIB

EL_OK, EL_INVALID_ARGUMENT, EL_RUNTIME_ERROR, EL_KV_OUT_OF_MEMORY, EL_LOGIC_ERROR, EL_CUDA_ERROR = 0, 1, 2, 3, 4, 6
TECH = {"softmax": 0, "state": 1, "classifier": 2, "never": 3, "always_at": 4, "fixed": 5}


class KvOutOfMemory(RuntimeError):
    """exitlab::KvOutOfMemory (kv_cache.hpp:101-103)."""


class LogicError(RuntimeError):
    """std::logic_error (e.g. decode_iteration on an empty batch)."""


class CudaError(RuntimeError):
    """Device failure (no reference counterpart)."""


_lib = None


def lib():
    """Load the in-tree library; raise (never fall back) when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"exitlab-b200 CUDA library not built: {LIB} (run __graft_entry__.build())")
        L = C.CDLL(LIB)
        L.el_last_error.restype = C.c_char_p
        L.el_engine_create.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
        L.el_engine_create_sized.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]
        L.el_engine_destroy.argtypes = [C.c_void_p]
        L.el_engine_set_option.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.el_engine_run.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.POINTER(C.c_void_p)]
        L.el_transcript_len.restype = C.c_int64
        L.el_transcript_len.argtypes = [C.c_void_p, C.c_char_p]
        L.el_transcript_get_i32.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
        L.el_transcript_get_f64.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
        L.el_transcript_kv.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int64]
        L.el_transcript_exit_states.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
        L.el_transcript_block_table.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
        L.el_transcript_free.argtypes = [C.c_void_p]
        L.el_transcript_free.restype = None
        L.el_session_begin.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_void_p]
        L.el_session_end.argtypes = [C.c_void_p]
        L.el_decode_iteration.argtypes = [C.c_void_p] + [C.c_void_p] * 5
        L.el_decode_run.argtypes = [C.c_void_p, C.c_int]
        L.el_decode_records.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 4
        L.el_decode_iterations_done.argtypes = [C.c_void_p]
        L.el_set_fixed_confidences.argtypes = [C.c_void_p, C.c_void_p]
        L.el_session_kv.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.el_session_cross_kv.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.el_session_hidden.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.el_session_block_table.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        L.el_time_decode.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_float)]
        L.el_time_kernel.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]
        L.el_sync.argtypes = [C.c_void_p]
        L.el_launches_per_iteration.argtypes = [C.c_void_p, C.c_int]
        L.el_plan_info.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        L.el_kv_block_trace.argtypes = [C.c_int] * 4 + [C.c_void_p] * 2 + [C.c_int, C.c_int, C.c_void_p]
        L.el_model_tensor.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64]
        L.el_set_device.argtypes = [C.c_int]
        L.el_device_count.argtypes = [C.c_void_p]
        L.el_transcript_metrics.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.el_metrics_compute.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int] + [C.c_void_p] * 9
        L.el_kv_allocate.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.el_kv_release.argtypes = [C.c_void_p, C.c_int]
        L.el_kv_append.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.el_kv_view.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.el_kv_commit.argtypes = [C.c_void_p, C.c_int]
        L.el_kv_lengths.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.el_kv_stats.argtypes = [C.c_void_p, C.c_void_p]
        L.el_layer_forward.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.el_kv_fill.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
        L.el_exit_confidence.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.el_greedy_tokens.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.el_sched_begin.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.el_sched_run.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_float)]
        L.el_sched_tokens.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
        L.el_sched_turns.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        _lib = L
    return _lib


def _check(rc: int):
    if rc == EL_OK:
        return
    msg = lib().el_last_error().decode()
    if rc == EL_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == EL_KV_OUT_OF_MEMORY:
        raise KvOutOfMemory(msg)
    if rc == EL_LOGIC_ERROR:
        raise LogicError(msg)
    if rc == EL_CUDA_ERROR:
        raise CudaError(msg)
    raise RuntimeError(msg)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- config types
@dataclass
class ModelConfig:  # model.hpp:18-25
    n_layers: int = 8
    d_model: int = 64
    vocab_size: int = 256
    seed: int = 0
    encoder_len: int = 0  # T5 mode (not in the reference): cross-attention over this many encoder states
    n_heads: int = 1  # extension: attention heads of d_model / n_heads features (the reference: 1)
    encoder_layers: int = 0  # T5 mode: a real encoder stack of this many layers (0: seeded encoder states)


@dataclass
class ExitTechnique:  # exit_policy.hpp:14-31
    kind: str = "never"
    exit_layer: int = 1

    @staticmethod
    def softmax_response():
        return ExitTechnique("softmax")

    @staticmethod
    def state_similarity():
        return ExitTechnique("state")

    @staticmethod
    def classifier():
        return ExitTechnique("classifier")

    @staticmethod
    def never():
        return ExitTechnique("never")

    @staticmethod
    def always_at(layer: int):
        return ExitTechnique("always_at", layer)

    @staticmethod
    def fixed():
        """test harness: injected confidences (el_set_fixed_confidences)."""
        return ExitTechnique("fixed")

    @property
    def name(self) -> str:  # technique_name (exit_policy.cpp:8-18)
        return f"always-at={self.exit_layer}" if self.kind == "always_at" else self.kind


def technique_from_name(name: str) -> ExitTechnique:  # exit_policy.cpp:20-36
    if name in ("softmax", "state", "classifier", "never"):
        return ExitTechnique(name)
    if name.startswith("always-at="):
        arg = name[len("always-at="):]
        if not arg.isdigit():
            raise ValueError(f"technique: bad layer in '{name}'")
        if int(arg) < 1:
            raise ValueError("technique: always-at layer must be >= 1")
        return ExitTechnique.always_at(int(arg))
    raise ValueError(f"technique: unknown name '{name}' (expected softmax|state|classifier|never|always-at=K)")


@dataclass
class ThresholdSchedule:  # exit_policy.hpp:36-42
    lambda0: float = 0.85
    gamma: float = 1.0
    lambda_min: float = 0.0


@dataclass
class CostModel:  # engine.hpp:18-28
    c_layer_fixed: float = 1e-3
    c_layer_per_seq: float = 1e-4
    c_fill_per_seq_layer: float = 2e-5
    c_check_softmax: float = 5e-5
    c_check_classifier: float = 5e-5
    c_check_state: float = 1e-5


@dataclass
class EngineConfig:  # engine.hpp:30-42
    model: ModelConfig = field(default_factory=ModelConfig)
    technique: ExitTechnique = field(default_factory=ExitTechnique.never)
    schedule: ThresholdSchedule = field(default_factory=ThresholdSchedule)
    costs: CostModel = field(default_factory=CostModel)
    max_batch: int = 8
    pool_blocks: int = 4096
    block_capacity: int = 16
    eos_token: int = 0
    capture_kv: bool = False
    synthetic_kv_seed: int = -1


class _CConfig(C.Structure):
    """el_engine_config (include/exitlab_b200.h); same layout as the oracle's."""
    _fields_ = [("n_layers", C.c_int), ("d_model", C.c_int), ("vocab_size", C.c_int),
                ("model_seed", C.c_uint64), ("technique", C.c_int), ("exit_layer", C.c_int),
                ("lambda0", C.c_double), ("gamma", C.c_double), ("lambda_min", C.c_double),
                ("c_layer_fixed", C.c_double), ("c_layer_per_seq", C.c_double),
                ("c_fill_per_seq_layer", C.c_double), ("c_check_softmax", C.c_double),
                ("c_check_classifier", C.c_double), ("c_check_state", C.c_double),
                ("max_batch", C.c_int), ("pool_blocks", C.c_int), ("block_capacity", C.c_int),
                ("eos_token", C.c_int), ("capture_kv", C.c_int), ("round_bf16", C.c_int),
                ("synthetic_kv_seed", C.c_int64), ("encoder_len", C.c_int), ("n_heads", C.c_int),
                ("encoder_layers", C.c_int)]


def to_c_config(cfg: EngineConfig) -> _CConfig:
    c = _CConfig()
    c.n_layers, c.d_model, c.vocab_size = cfg.model.n_layers, cfg.model.d_model, cfg.model.vocab_size
    c.model_seed = cfg.model.seed
    c.technique = TECH[cfg.technique.kind]
    c.exit_layer = cfg.technique.exit_layer
    c.lambda0, c.gamma, c.lambda_min = cfg.schedule.lambda0, cfg.schedule.gamma, cfg.schedule.lambda_min
    for k in ("c_layer_fixed", "c_layer_per_seq", "c_fill_per_seq_layer", "c_check_softmax",
              "c_check_classifier", "c_check_state"):
        setattr(c, k, getattr(cfg.costs, k))
    c.max_batch, c.pool_blocks, c.block_capacity, c.eos_token = (cfg.max_batch, cfg.pool_blocks,
                                                                  cfg.block_capacity, cfg.eos_token)
    c.capture_kv = int(cfg.capture_kv)
    c.round_bf16 = 1
    c.synthetic_kv_seed = cfg.synthetic_kv_seed
    c.encoder_len = cfg.model.encoder_len
    c.n_heads = cfg.model.n_heads
    c.encoder_layers = cfg.model.encoder_layers
    return c


# ---------------------------------------------------------------- workload
@dataclass
class Request:  # workload.hpp:10-14
    arrival_time: float
    prompt: list
    max_new_tokens: int = 1


@dataclass
class Workload:
    requests: list = field(default_factory=list)

    def flat(self):
        n = len(self.requests)
        arrival = np.array([r.arrival_time for r in self.requests], dtype=np.float64)
        off = np.zeros(n + 1, dtype=np.int32)
        toks = []
        for i, r in enumerate(self.requests):
            toks.extend(int(t) for t in r.prompt)
            off[i + 1] = len(toks)
        return (arrival, off, np.array(toks, dtype=np.int32),
                np.array([r.max_new_tokens for r in self.requests], dtype=np.int32))

    @staticmethod
    def from_flat(arrival, off, prompt, max_new):
        return Workload([Request(float(arrival[i]), prompt[off[i]:off[i + 1]].tolist(), int(max_new[i]))
                         for i in range(len(arrival))])


# ---------------------------------------------------------------- transcript
I32_FIELDS = ["pf_seq", "pf_positions", "it_output_layer", "it_batch_off", "ps_seq", "ps_accept",
              "ps_token", "sq_id", "sq_max_new", "sq_prompt_off", "sq_prompt", "sq_tok_off",
              "sq_tokens", "sq_exit_layers", "sq_iter_out"]
F64_FIELDS = ["pf_clock", "pf_charge", "it_clock", "it_charge", "sq_arrival", "sq_first",
              "sq_finish", "meta", "it_conf"]


class Transcript:
    """Flat transcript (engine.hpp:67-123), fields identical to the oracle's."""

    def __init__(self, handle, d, L):
        L_ = lib()
        self.f = {}
        for name in I32_FIELDS:
            n = L_.el_transcript_len(handle, name.encode())
            a = np.zeros(max(n, 0), dtype=np.int32)
            if n > 0:
                _check(L_.el_transcript_get_i32(handle, name.encode(), _ptr(a)))
            self.f[name] = a
        for name in F64_FIELDS:
            n = L_.el_transcript_len(handle, name.encode())
            a = np.zeros(max(n, 0), dtype=np.float64)
            if n > 0:
                _check(L_.el_transcript_get_f64(handle, name.encode(), _ptr(a)))
            self.f[name] = a
        self._h = handle
        self.d, self.L = d, L

    def __del__(self):
        try:
            if self._h:
                lib().el_transcript_free(self._h)
        except Exception:
            pass

    def __getitem__(self, k):
        return self.f[k]

    @property
    def final_clock(self):
        return float(self.f["meta"][0])

    @property
    def iterations(self):
        off = self.f["it_batch_off"]
        return [dict(clock=self.f["it_clock"][i], charge=self.f["it_charge"][i],
                     output_layer=int(self.f["it_output_layer"][i]),
                     batch_ids=self.f["ps_seq"][off[i]:off[i + 1]].tolist(),
                     accept=self.f["ps_accept"][off[i]:off[i + 1]].tolist(),
                     tokens=self.f["ps_token"][off[i]:off[i + 1]].tolist())
                for i in range(len(self.f["it_output_layer"]))]

    @property
    def sequences(self):
        po, to = self.f["sq_prompt_off"], self.f["sq_tok_off"]
        return [dict(id=int(self.f["sq_id"][i]), arrival=self.f["sq_arrival"][i],
                     first_token=self.f["sq_first"][i], finish=self.f["sq_finish"][i],
                     max_new=int(self.f["sq_max_new"][i]),
                     prompt=self.f["sq_prompt"][po[i]:po[i + 1]].tolist(),
                     tokens=self.f["sq_tokens"][to[i]:to[i + 1]].tolist(),
                     exit_layers=self.f["sq_exit_layers"][to[i]:to[i + 1]].tolist(),
                     iter_output_layers=self.f["sq_iter_out"][to[i]:to[i + 1]].tolist())
                for i in range(len(self.f["sq_id"]))]

    # ---- persistence: the reference's JSON-lines format (engine.cpp:336-393) ----
    def to_jsonl(self, path, model: "ModelConfig" = None, technique: "ExitTechnique" = None):
        """write_transcript_jsonl: same records, key order and number formatting as the
        reference (nlohmann ordered_json dump), so B200 transcripts are byte-comparable with
        the reference's and readable by read_transcript_jsonl / compute_metrics."""
        write_transcript_jsonl(self, path, model or self.model, technique or self.technique)

    def kv(self, seq_id, layer):
        n = 1 << 22
        k = np.zeros(n)
        v = np.zeros(n)
        c = lib().el_transcript_kv(self._h, seq_id, layer, _ptr(k), _ptr(v), n)
        if c < 0:
            _check(-c)
        return k[: c * self.d].reshape(c, self.d), v[: c * self.d].reshape(c, self.d)

    def block_table(self, seq_id):
        """capture_kv: the device block table [L][bpl] of the sequence at eviction"""
        out = np.zeros(1 << 20, np.int32)
        n = lib().el_transcript_block_table(self._h, seq_id, _ptr(out), out.size)
        if n < 0:
            _check(-n)
        return out[: self.L * n].reshape(self.L, n)

    def exit_states(self, seq_id):
        n = 1 << 22
        o = np.zeros(n)
        c = lib().el_transcript_exit_states(self._h, seq_id, _ptr(o), n)
        if c < 0:
            _check(-c)
        return o[: c * self.d].reshape(c, self.d)


def _json_num(x):
    if isinstance(x, (bool, np.bool_)):
        return "true" if x else "false"
    if isinstance(x, (int, np.integer)):
        return str(int(x))
    x = float(x)
    if x != x or x in (float("inf"), float("-inf")):
        return "null"  # nlohmann dumps non-finite numbers as null
    r = repr(x)  # shortest round-trip, like nlohmann's dtoa
    if "e" not in r and "." not in r:
        r += ".0"
    return r


def _json_dump(v):
    """nlohmann::ordered_json::dump() formatting: no spaces, insertion order."""
    import json
    if isinstance(v, dict):
        return "{" + ",".join(json.dumps(k) + ":" + _json_dump(x) for k, x in v.items()) + "}"
    if isinstance(v, (list, tuple)):
        return "[" + ",".join(_json_dump(x) for x in v) + "]"
    if isinstance(v, str):
        return json.dumps(v, ensure_ascii=False)
    return _json_num(v)


def transcript_records(t, model, technique):
    """The records of write_transcript_jsonl (engine.cpp:336-393) for a flat transcript."""
    m = t["meta"]  # final_clock, total_idle, pool_blocks, free_blocks, peak_blocks
    yield {"type": "meta", "n_layers": model.n_layers, "d_model": model.d_model, "vocab_size": model.vocab_size,
           "model_seed": int(model.seed), "technique": technique.name, "final_clock": float(m[0]),
           "total_idle": float(m[1]),
           "cache": {"pool_blocks": int(m[2]), "free_blocks": int(m[3]), "peak_blocks": int(m[4])}}
    for i in range(len(t["pf_seq"])):
        yield {"type": "prefill", "clock": float(t["pf_clock"][i]), "charge": float(t["pf_charge"][i]),
               "seq_id": int(t["pf_seq"][i]), "positions": int(t["pf_positions"][i])}
    for it in t.iterations:
        yield {"type": "iteration", "clock": float(it["clock"]), "charge": float(it["charge"]),
               "batch_ids": [int(x) for x in it["batch_ids"]], "output_layer": it["output_layer"],
               "per_seq": [{"seq_id": int(sid), "accept_layer": int(a), "token": int(tok)}
                           for sid, a, tok in zip(it["batch_ids"], it["accept"], it["tokens"])]}
    for sq in t.sequences:
        yield {"type": "sequence", "seq_id": sq["id"], "arrival": float(sq["arrival"]),
               "first_token": float(sq["first_token"]), "finish": float(sq["finish"]),
               "max_new_tokens": sq["max_new"], "prompt": sq["prompt"], "tokens": sq["tokens"],
               "exit_layers": sq["exit_layers"], "iter_output_layers": sq["iter_output_layers"]}


def write_transcript_jsonl(t, path, model, technique):
    """write_transcript_jsonl (engine.cpp:336-393) for any flat transcript (product, oracle port or
    reference wrapper): byte-identical to the reference's writer."""
    with open(path, "w") as f:
        for rec in transcript_records(t, model, technique):
            f.write(_json_dump(rec) + "\n")


def read_transcript_jsonl(path):
    """read_transcript_jsonl (engine.cpp:395-461): the records as dicts, validated like the
    reference (unknown types and a missing meta record are errors)."""
    import json
    out = {"meta": None, "prefills": [], "iterations": [], "sequences": []}
    with open(path) as f:
        for no, line in enumerate(f, 1):
            if not line.strip():
                continue
            try:
                j = json.loads(line)
            except json.JSONDecodeError as e:
                raise RuntimeError(f"transcript: parse error at line {no}: {e}") from None
            kind = j.get("type")
            if kind == "meta":
                out["meta"] = j
            elif kind in ("prefill", "iteration", "sequence"):
                out[kind + "s" if kind != "prefill" else "prefills"].append(j)
            else:
                raise RuntimeError(f"transcript: unknown record type '{kind}' at line {no}")
    if out["meta"] is None:
        raise RuntimeError(f"transcript: missing meta record in {path}")
    return out


# ---------------------------------------------------------------- metrics (metrics.hpp:20-45)
class _CMetrics(C.Structure):
    _fields_ = [("throughput", C.c_double), ("inner_token_latency", C.c_double), ("early_exit_rate_pct", C.c_double),
                ("mean_layers_per_token", C.c_double), ("total_sim_time", C.c_double),
                ("total_idle_time", C.c_double), ("wall_clock_info_s", C.c_double), ("total_tokens", C.c_int64),
                ("iterations", C.c_int64), ("n_layers", C.c_int), ("pool_blocks", C.c_int),
                ("free_blocks", C.c_int), ("peak_blocks", C.c_int)]


@dataclass
class MetricsReport:
    """MetricsReport (metrics.hpp:20-34)."""
    throughput: float = 0.0
    inner_token_latency: float = 0.0
    early_exit_rate_pct: float = 0.0
    exit_layer_histogram: list = field(default_factory=list)
    accept_layer_histogram: list = field(default_factory=list)
    mean_layers_per_token: float = 0.0
    total_sim_time: float = 0.0
    total_idle_time: float = 0.0
    total_tokens: int = 0
    iterations: int = 0
    n_layers: int = 0
    cache: dict = field(default_factory=lambda: {"pool_blocks": 0, "free_blocks": 0, "peak_blocks": 0})
    wall_clock_info_s: float = 0.0


def _metrics_from_c(m, eh, ah):
    return MetricsReport(m.throughput, m.inner_token_latency, m.early_exit_rate_pct, eh.tolist(), ah.tolist(),
                         m.mean_layers_per_token, m.total_sim_time, m.total_idle_time, int(m.total_tokens),
                         int(m.iterations), int(m.n_layers),
                         {"pool_blocks": m.pool_blocks, "free_blocks": m.free_blocks, "peak_blocks": m.peak_blocks},
                         m.wall_clock_info_s)


def compute_metrics(t, n_layers=None) -> MetricsReport:
    """compute_metrics (metrics.cpp:13-58) -- native (libexitlab_b200) over any flat transcript:
    this engine's Transcript, or the oracle's / reference's (then pass n_layers)."""
    L = n_layers or t.L
    m = _CMetrics()
    eh = np.zeros(L, np.int64)
    ah = np.zeros(L, np.int64)
    if isinstance(t, Transcript):
        _check(lib().el_transcript_metrics(t._h, C.byref(m), _ptr(eh), _ptr(ah)))
    else:
        f = {k: np.ascontiguousarray(t[k]) for k in ("it_output_layer", "it_batch_off", "sq_id", "sq_tok_off",
                                                     "sq_exit_layers", "sq_first", "sq_finish", "meta")}
        _check(lib().el_metrics_compute(L, len(f["it_output_layer"]), _ptr(f["it_output_layer"].astype(np.int32)),
                                        _ptr(f["it_batch_off"].astype(np.int32)), len(f["sq_id"]),
                                        _ptr(f["sq_id"].astype(np.int32)), _ptr(f["sq_tok_off"].astype(np.int32)),
                                        _ptr(f["sq_exit_layers"].astype(np.int32)),
                                        _ptr(f["sq_first"].astype(np.float64)), _ptr(f["sq_finish"].astype(np.float64)),
                                        _ptr(f["meta"].astype(np.float64)), C.byref(m), _ptr(eh), _ptr(ah)))
    return _metrics_from_c(m, eh, ah)


def session_metrics(output_layers, accept, n_layers) -> dict:
    """compute_metrics' token-weighted exit statistics for fixed-batch decode records
    (every iteration decodes the whole batch): early-exit rate, mean layers per token and the
    exit / accept histograms (metrics.cpp:33-55)."""
    e = np.asarray(output_layers, np.int64)
    a = np.asarray(accept, np.int64).reshape(len(e), -1)
    B = a.shape[1]
    return {"early_exit_rate_pct": float(100.0 * np.mean(e < n_layers)) if len(e) else 0.0,
            "mean_layers_per_token": float(e.mean()) if len(e) else 0.0,
            "exit_layer_histogram": (np.bincount(e - 1, minlength=n_layers) * B).tolist(),
            "accept_layer_histogram": np.bincount(a.ravel() - 1, minlength=n_layers).tolist()}


def _json_pretty(v, ind=0):
    """nlohmann::ordered_json::dump(2) formatting of the report object."""
    import json
    pad, pad2 = " " * ind, " " * (ind + 2)
    if isinstance(v, dict):
        if not v:
            return "{}"
        return "{\n" + ",\n".join(pad2 + json.dumps(k) + ": " + _json_pretty(x, ind + 2) for k, x in v.items()) + \
            "\n" + pad + "}"
    return _json_dump(v)  # arrays stay on one line in this nlohmann build (observed, tests/test_metrics_cpu.py)


def _g17(x):
    return "%.17g" % float(x)


def write_report(r: MetricsReport, path, fmt):
    """write_report (metrics.cpp:178-195): JSON (ordered keys, dump(2)) or CSV (metric,value with
    %.17g doubles), byte-identical to the reference's writer."""
    if fmt not in ("json", "csv"):
        raise ValueError(f"write_report: unsupported format '{fmt}' (expected json or csv)")
    if fmt == "json":
        j = {"throughput_tokens_per_s": float(r.throughput), "inner_token_latency_s": float(r.inner_token_latency),
             "early_exit_rate_pct": float(r.early_exit_rate_pct),
             "exit_layer_histogram": [int(x) for x in r.exit_layer_histogram],
             "accept_layer_histogram": [int(x) for x in r.accept_layer_histogram],
             "mean_layers_per_token": float(r.mean_layers_per_token), "total_sim_time_s": float(r.total_sim_time),
             "total_idle_time_s": float(r.total_idle_time), "total_tokens": int(r.total_tokens),
             "iterations": int(r.iterations), "n_layers": int(r.n_layers),
             "cache": {"pool_blocks": int(r.cache["pool_blocks"]), "free_blocks": int(r.cache["free_blocks"]),
                       "peak_blocks": int(r.cache["peak_blocks"])},
             "wall_clock_info_s": float(r.wall_clock_info_s)}
        text = _json_pretty(j) + "\n"
    else:
        rows = [("throughput_tokens_per_s", _g17(r.throughput)), ("inner_token_latency_s", _g17(r.inner_token_latency)),
                ("early_exit_rate_pct", _g17(r.early_exit_rate_pct)),
                ("mean_layers_per_token", _g17(r.mean_layers_per_token)), ("total_sim_time_s", _g17(r.total_sim_time)),
                ("total_idle_time_s", _g17(r.total_idle_time)), ("total_tokens", str(int(r.total_tokens))),
                ("iterations", str(int(r.iterations))), ("n_layers", str(int(r.n_layers))),
                ("cache_pool_blocks", str(int(r.cache["pool_blocks"]))),
                ("cache_free_blocks", str(int(r.cache["free_blocks"]))),
                ("cache_peak_blocks", str(int(r.cache["peak_blocks"]))),
                ("wall_clock_info_s", _g17(r.wall_clock_info_s))]
        rows += [(f"exit_layer_{i + 1}", str(int(x))) for i, x in enumerate(r.exit_layer_histogram)]
        rows += [(f"accept_layer_{i + 1}", str(int(x))) for i, x in enumerate(r.accept_layer_histogram)]
        text = "metric,value\n" + "".join(f"{k},{v}\n" for k, v in rows)
    with open(path, "w") as f:
        f.write(text)


def read_report(path, fmt) -> MetricsReport:
    """read_report (metrics.cpp:197-210): the inverse of write_report, reference error messages."""
    import json
    if fmt not in ("json", "csv"):
        raise ValueError(f"read_report: unsupported format '{fmt}'")
    if not os.path.exists(path):
        raise RuntimeError(f"read_report: cannot open {path}")
    if fmt == "json":
        try:
            with open(path) as f:
                j = json.load(f)
        except json.JSONDecodeError as e:
            raise ValueError(f"report: {path}: {e}") from None
        try:
            return MetricsReport(float(j["throughput_tokens_per_s"]), float(j["inner_token_latency_s"]),
                                 float(j["early_exit_rate_pct"]), [int(x) for x in j["exit_layer_histogram"]],
                                 [int(x) for x in j["accept_layer_histogram"]], float(j["mean_layers_per_token"]),
                                 float(j["total_sim_time_s"]), float(j["total_idle_time_s"]), int(j["total_tokens"]),
                                 int(j["iterations"]), int(j["n_layers"]),
                                 {k: int(j["cache"][k]) for k in ("pool_blocks", "free_blocks", "peak_blocks")},
                                 float(j["wall_clock_info_s"]))
        except KeyError as e:
            raise ValueError(f"report: {path}: missing key {e}") from None
    with open(path) as f:
        lines = f.read().split("\n")
    if not lines or lines[0] != "metric,value":
        raise ValueError(f"report: {path}: missing 'metric,value' header")
    rows = {}
    for line in lines[1:]:
        if not line:
            continue
        if "," not in line:
            raise ValueError(f"report: {path}: bad row '{line}'")
        k, v = line.split(",", 1)
        rows.setdefault(k, v)

    def take(k):
        if k not in rows:
            raise ValueError(f"report: {path}: missing metric '{k}'")
        return rows[k]
    n = int(take("n_layers"))
    return MetricsReport(float(take("throughput_tokens_per_s")), float(take("inner_token_latency_s")),
                         float(take("early_exit_rate_pct")), [int(take(f"exit_layer_{i}")) for i in range(1, n + 1)],
                         [int(take(f"accept_layer_{i}")) for i in range(1, n + 1)],
                         float(take("mean_layers_per_token")), float(take("total_sim_time_s")),
                         float(take("total_idle_time_s")), int(take("total_tokens")), int(take("iterations")), n,
                         {"pool_blocks": int(take("cache_pool_blocks")), "free_blocks": int(take("cache_free_blocks")),
                          "peak_blocks": int(take("cache_peak_blocks"))}, float(take("wall_clock_info_s")))


# ---------------------------------------------------------------- engine
class Engine:
    """exitlab::Engine on one B200 (engine.hpp:131-147). Weights are seeded from
    config.model (ModelWeights::seeded, model.cpp:37-59) and stored as bf16."""

    def __init__(self, config: EngineConfig, graph: bool = True, mega=None):
        """graph/mega select how a decode iteration is launched: mega=True = one
        persistent kernel per iteration (layer loop on the device); mega=False =
        per-phase kernels in a CUDA graph with a device-side WHILE (graph) or a
        host-driven layer loop (eager); mega=None (default) picks per batch size
        (persistent at batch >= 128, where it measured faster)."""
        self.config = config
        self._c = to_c_config(config)
        h = C.c_void_p()
        _check(lib().el_engine_create_sized(C.byref(self._c), C.sizeof(self._c), C.byref(h)))
        self._h = h
        self.L, self.d, self.V = config.model.n_layers, config.model.d_model, config.model.vocab_size
        self.B = 0
        self.set_option("graph", int(graph))
        self.set_option("mega", 2 if mega is None else int(bool(mega)))

    def close(self):
        if getattr(self, "_h", None):
            lib().el_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key: str, value: int):
        _check(lib().el_engine_set_option(self._h, key.encode(), int(value)))

    def run(self, workload: Workload) -> Transcript:  # Engine::run (engine.cpp:110-330)
        arrival, off, prompt, max_new = workload.flat()
        t = C.c_void_p()
        _check(lib().el_engine_run(self._h, len(arrival), _ptr(arrival), _ptr(off), _ptr(prompt),
                                   _ptr(max_new), C.byref(t)))
        tr = Transcript(t, self.d, self.L)
        tr.model, tr.technique = self.config.model, self.config.technique
        return tr

    # ---- fixed-batch decode session over a seeded KV prefix ----
    def session_begin(self, first_tokens, prefix_len, capacity, kv_seed, seq_ids=None):
        ft = np.ascontiguousarray(first_tokens, dtype=np.int32)
        ids = None if seq_ids is None else np.ascontiguousarray(seq_ids, dtype=np.int32)
        _check(lib().el_session_begin(self._h, len(ft), _ptr(ft), prefix_len, capacity, kv_seed, _ptr(ids)))
        self.B = len(ft)

    def session_end(self):
        _check(lib().el_session_end(self._h))

    def decode_iteration(self, tokens_in=None):
        """decode_iteration (engine.cpp:208-310) with host buffers in and out."""
        B, L = self.B, self.L
        tin = None if tokens_in is None else np.ascontiguousarray(tokens_in, dtype=np.int32)
        tok = np.zeros(B, np.int32)
        acc = np.zeros(B, np.int32)
        conf = np.zeros((L, B), np.float32)
        e = np.zeros(1, np.int32)
        _check(lib().el_decode_iteration(self._h, _ptr(tin), _ptr(tok), _ptr(acc), _ptr(conf), _ptr(e)))
        return dict(output_layer=int(e[0]), tokens=tok, accept=acc, conf=conf)

    def decode_run(self, n):
        _check(lib().el_decode_run(self._h, n))

    def records(self, first, n):
        B, L = self.B, self.L
        tok = np.zeros((n, B), np.int32)
        acc = np.zeros((n, B), np.int32)
        out = np.zeros(n, np.int32)
        conf = np.zeros((n, L, B), np.float32)
        _check(lib().el_decode_records(self._h, first, n, _ptr(tok), _ptr(acc), _ptr(out), _ptr(conf)))
        return dict(tokens=tok, accept=acc, output_layer=out, conf=conf)

    def set_fixed_confidences(self, conf):
        c = np.ascontiguousarray(conf, dtype=np.float32)
        _check(lib().el_set_fixed_confidences(self._h, _ptr(c)))

    def kv(self, row, layer, pos):
        k = np.zeros(self.d, np.float32)
        v = np.zeros(self.d, np.float32)
        _check(lib().el_session_kv(self._h, row, layer, pos, _ptr(k), _ptr(v)))
        return k, v

    def cross_kv(self, row, layer):
        """T5 mode: the row's static cross K/V at `layer` ([encoder_len][d] each)"""
        T = self.config.model.encoder_len
        k = np.zeros((T, self.d), np.float32)
        v = np.zeros((T, self.d), np.float32)
        _check(lib().el_session_cross_kv(self._h, row, layer, _ptr(k), _ptr(v)))
        return k, v

    def hidden(self, parity):
        out = np.zeros((self.B, self.d), np.float32)
        _check(lib().el_session_hidden(self._h, parity, _ptr(out)))
        return out

    def block_table(self, row, bpl_cap=4096):
        out = np.zeros(self.L * bpl_cap, np.int32)
        n = lib().el_session_block_table(self._h, row, _ptr(out), bpl_cap)
        if n < 0:
            _check(-n)
        return out[: self.L * n].reshape(self.L, n)

    def time_decode(self, n):
        ms = C.c_float()
        _check(lib().el_time_decode(self._h, n, C.byref(ms)))
        return ms.value

    def time_kernel(self, kind, layer, reps):
        ms = C.c_float()
        _check(lib().el_time_kernel(self._h, kind, layer, reps, C.byref(ms)))
        return ms.value

    def sync(self):
        _check(lib().el_sync(self._h))

    def launches_per_iteration(self, output_layer):
        return lib().el_launches_per_iteration(self._h, output_layer)

    def plan_info(self):
        out = np.zeros(64, np.int64)
        n = lib().el_plan_info(self._h, _ptr(out), 64)
        names = ["attn_cb", "attn_stages", "attn_max_chunks", "n_pad", "qkv_splits", "wo_splits", "up_splits",
                 "down_splits", "fill_splits", "qkv_stages", "lm_tiles", "dp", "fp", "Vp", "bpl_max",
                 "mega_qkv_mode", "mega_wo_mode", "mega_up_mode", "mega_qkv_splits", "mega_wo_splits",
                 "mega_up_splits", "mega_down_splits", "mega_fill_splits", "mega_qkv_nt", "mega_wo_nt", "mega_up_nt",
                 "mega_stages", "mega_stages2", "mega_att_stages", "mega", "pipe", "lm_pair", "lm_keep", "lm_tail_tr", "lm_stages"]
        return dict(zip(names, out[:n].tolist()))

    # ---- layer-level scheduling over the session's batch ----
    def sched_begin(self, policy="greedy", M=None):
        """Switch the (fresh) session to layer-level scheduling: turns run one layer for the
        sequences whose next layer it is, each exiting on its own accept.  policy "greedy"
        (greedy_action) or "linear" (argmax_a M[a].v, LinearQ; M = L x L)."""
        pol = {"greedy": 0, "linear": 1}[policy]
        m = None if M is None else np.ascontiguousarray(M, dtype=np.float64).reshape(self.L, self.L)
        _check(lib().el_sched_begin(self._h, pol, _ptr(m)))

    def sched_run(self, n_turns):
        """run n turns; returns their elapsed milliseconds (CUDA events, host round trips included)"""
        ms = C.c_float()
        _check(lib().el_sched_run(self._h, int(n_turns), C.byref(ms)))
        return ms.value

    def sched_tokens(self, row):
        n = lib().el_sched_tokens(self._h, int(row), None, None, 0)
        if n < 0:
            _check(-n)
        t = np.zeros(max(n, 1), np.int32)
        x = np.zeros(max(n, 1), np.int32)
        lib().el_sched_tokens(self._h, int(row), _ptr(t), _ptr(x), n)
        return t[:n], x[:n]

    def sched_turns(self):
        n = lib().el_sched_turns(self._h, None, None, 0)
        if n < 0:
            _check(-n)
        a = np.zeros(max(n, 1), np.int32)
        r = np.zeros(max(n, 1), np.int32)
        lib().el_sched_turns(self._h, _ptr(a), _ptr(r), n)
        return a[:n], r[:n]

    def kv_store(self) -> "KvStore":
        """the device pool as a KvStore (sub-engine API; reset by run() / session_begin())"""
        return KvStore(self)

    def model_tensor(self, which, layer=0):
        names = {"embedding": 0, "lm_head": 1, "probe_w": 2, "probe_b": 3, "w_q": 4, "w_k": 5, "w_v": 6,
                 "w_o": 7, "w_up": 8, "w_down": 9}
        w = names[which] if isinstance(which, str) else which
        d, V = self.d, self.V
        shape = {0: (V, d), 1: (V, d), 2: (d,), 3: (1,), 4: (d, d), 5: (d, d), 6: (d, d), 7: (d, d),
                 8: (4 * d, d), 9: (d, 4 * d)}[w]
        out = np.zeros(int(np.prod(shape)), np.uint16)
        _check(lib().el_model_tensor(self._h, w, layer, _ptr(out), out.size))
        return out.reshape(shape)


def set_device(device: int):
    """Device for engines created afterwards in this thread (one process per GPU)."""
    _check(lib().el_set_device(int(device)))


def device_count() -> int:
    n = C.c_int(0)
    _check(lib().el_device_count(C.byref(n)))
    return n.value


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def kv_block_trace(n_layers, pool, cap, ops, caps, n_ids, bpl_max):
    """KvStore LIFO allocation order on the host mirror (kv_cache.cpp:53-55, 78-106, 182-194)."""
    ops = np.ascontiguousarray(ops, dtype=np.int32)
    caps = np.ascontiguousarray(caps, dtype=np.int32)
    tab = np.zeros((n_ids, n_layers, bpl_max), np.int32)
    nf = lib().el_kv_block_trace(n_layers, pool, cap, len(ops), _ptr(ops), _ptr(caps), n_ids, bpl_max, _ptr(tab))
    if nf < 0:
        _check(-nf)
    return tab, nf


# ---------------------------------------------------------------- sub-engine API (device pool)
def _f32(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a if shape is None else a.reshape(shape)


class KvStore:
    """KvStore (kv_cache.hpp:45-75) on an Engine's device pool: the same LIFO block order,
    write-once / contiguity / capacity / commit-completeness checks and exception classes
    (ValueError = std::invalid_argument, RuntimeError = std::runtime_error, KvOutOfMemory).
    Values are stored in bf16 (the engine's K/V precision)."""

    def __init__(self, engine: "Engine"):
        self.e = engine

    def allocate(self, seq_id, capacity_tokens):
        _check(lib().el_kv_allocate(self.e._h, int(seq_id), int(capacity_tokens)))

    def append(self, seq_id, layer, position, k, v):
        d = self.e.d
        _check(lib().el_kv_append(self.e._h, int(seq_id), int(layer), int(position), _ptr(_f32(k, (d,))),
                                  _ptr(_f32(v, (d,)))))

    def view(self, seq_id, layer, upto_position):
        d = self.e.d
        k = np.zeros((max(int(upto_position), 0), d), np.float32)
        v = np.zeros_like(k)
        _check(lib().el_kv_view(self.e._h, int(seq_id), int(layer), int(upto_position), _ptr(k), _ptr(v)))
        return k, v

    def commit(self, seq_id):
        _check(lib().el_kv_commit(self.e._h, int(seq_id)))

    def release(self, seq_id):
        _check(lib().el_kv_release(self.e._h, int(seq_id)))

    def committed_len(self, seq_id):
        c = np.zeros(1, np.int32)
        _check(lib().el_kv_lengths(self.e._h, int(seq_id), _ptr(c), None))
        return int(c[0])

    def written_len(self, seq_id, layer):
        w = np.zeros(self.e.L, np.int32)
        _check(lib().el_kv_lengths(self.e._h, int(seq_id), None, _ptr(w)))
        if not 1 <= layer <= self.e.L:
            raise ValueError("written_len: layer out of range")
        return int(w[layer - 1])

    def stats(self):
        o = np.zeros(4, np.int32)
        _check(lib().el_kv_stats(self.e._h, _ptr(o)))
        return {"pool_blocks": int(o[0]), "free_blocks": int(o[1]), "peak_blocks_in_use": int(o[2]),
                "sequences": int(o[3])}


def _batch(batch, d):
    ids = np.ascontiguousarray([int(s) for s, _ in batch], dtype=np.int32)
    h = _f32(np.stack([np.asarray(x, np.float32).reshape(d) for _, x in batch]))
    return ids, h


def layer_forward(engine: "Engine", layer, batch):
    """layer_forward(weights, layer, batch, cache) (model.hpp:64-66) on the device: batch =
    [(seq_id, h)], K/V appended to engine.kv_store() at each sequence's committed length."""
    ids, h = _batch(batch, engine.d)
    out = np.zeros_like(h)
    _check(lib().el_layer_forward(engine._h, int(layer), len(ids), _ptr(ids), _ptr(h), _ptr(out)))
    return [out[i] for i in range(len(ids))]


def fill_skipped(engine: "Engine", batch, output_layer):
    """fill_skipped(cache, batch, output_layer, compute_kv_pair) (kv_cache.hpp:107-115): K/V of the
    layers after output_layer projected from each exit state, one grouped GEMM on the device."""
    ids, h = _batch(batch, engine.d)
    _check(lib().el_kv_fill(engine._h, len(ids), _ptr(ids), _ptr(h), int(output_layer)))


def exit_confidence(engine: "Engine", layer, h_cur, h_prev=None):
    """The engine technique's confidence (exit_policy.hpp:46-70) for states h_cur [n][d] (h_prev for
    state similarity) and decide's strict '>' against threshold_at(layer); returns (conf, accept)."""
    hc = _f32(np.atleast_2d(h_cur))
    hp = None if h_prev is None else _f32(np.atleast_2d(h_prev))
    n = hc.shape[0]
    conf = np.zeros(n, np.float32)
    acc = np.zeros(n, np.int32)
    _check(lib().el_exit_confidence(engine._h, int(layer), n, _ptr(hp), _ptr(hc), _ptr(conf), _ptr(acc)))
    return conf, acc.astype(bool)


def greedy_tokens(engine: "Engine", h):
    """greedy_token(lm_head_logits(h)) (model.hpp:71-76) for states h [n][d]."""
    hh = _f32(np.atleast_2d(h))
    out = np.zeros(hh.shape[0], np.int32)
    _check(lib().el_greedy_tokens(engine._h, hh.shape[0], _ptr(hh), _ptr(out)))
    return out
