"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the two CPU checkers.

* ``Port``  -> oracle/liboracle.so, the C restatement (exitlab_oracle.c)
* ``Ref``   -> oracle/_ref/libexitlab_ref.so, the unmodified reference sources
               (/root/reference/proj/src) + the C-ABI shim ref_capi.cpp

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg import this module.  The product package never does.
Both libraries expose the same flat transcript layout as the product, so
``Transcript`` objects from any of the three compare field by field.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libexitlab_ref.so")
REF_SRC = "/root/reference/proj"

TECH = {"softmax": 0, "state": 1, "classifier": 2, "never": 3, "always_at": 4, "fixed": 5}

I32_FIELDS = ["pf_seq", "pf_positions", "it_output_layer", "it_batch_off", "ps_seq", "ps_accept",
              "ps_token", "sq_id", "sq_max_new", "sq_prompt_off", "sq_prompt", "sq_tok_off",
              "sq_tokens", "sq_exit_layers", "sq_iter_out"]
F64_FIELDS = ["pf_clock", "pf_charge", "it_clock", "it_charge", "sq_arrival", "sq_first",
              "sq_finish", "meta", "it_conf"]


def build(quiet: bool = True) -> None:
    """make the port (always) and _ref (only where /root/reference exists)."""
    targets = ["liboracle.so"] + (["ref"] if os.path.isdir(REF_SRC) else [])
    out = subprocess.run(["make", "-C", HERE, "-j8"] + [os.path.join(HERE, t) if t.endswith(".so") else t
                                                        for t in targets],
                         capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


class EngineConfig(C.Structure):
    """Layout of eo_engine_config (exitlab_oracle.h)."""
    _fields_ = [("n_layers", C.c_int), ("d_model", C.c_int), ("vocab_size", C.c_int),
                ("model_seed", C.c_uint64), ("technique", C.c_int), ("exit_layer", C.c_int),
                ("lambda0", C.c_double), ("gamma", C.c_double), ("lambda_min", C.c_double),
                ("c_layer_fixed", C.c_double), ("c_layer_per_seq", C.c_double),
                ("c_fill_per_seq_layer", C.c_double), ("c_check_softmax", C.c_double),
                ("c_check_classifier", C.c_double), ("c_check_state", C.c_double),
                ("max_batch", C.c_int), ("pool_blocks", C.c_int), ("block_capacity", C.c_int),
                ("eos_token", C.c_int), ("capture_kv", C.c_int), ("round_bf16", C.c_int),
                ("synthetic_kv_seed", C.c_int64)]


def engine_config(n_layers=8, d_model=64, vocab_size=256, model_seed=0, technique="never",
                  exit_layer=1, lambda0=0.85, gamma=1.0, lambda_min=0.0, max_batch=8,
                  pool_blocks=4096, block_capacity=16, eos_token=0, capture_kv=False,
                  round_bf16=False, synthetic_kv_seed=-1, costs=None) -> EngineConfig:
    c = EngineConfig()
    c.n_layers, c.d_model, c.vocab_size, c.model_seed = n_layers, d_model, vocab_size, model_seed
    c.technique = TECH[technique] if isinstance(technique, str) else int(technique)
    c.exit_layer = exit_layer
    c.lambda0, c.gamma, c.lambda_min = lambda0, gamma, lambda_min
    cm = dict(c_layer_fixed=1e-3, c_layer_per_seq=1e-4, c_fill_per_seq_layer=2e-5,
              c_check_softmax=5e-5, c_check_classifier=5e-5, c_check_state=1e-5)
    cm.update(costs or {})
    for k, v in cm.items():
        setattr(c, k, v)
    c.max_batch, c.pool_blocks, c.block_capacity, c.eos_token = max_batch, pool_blocks, block_capacity, eos_token
    c.capture_kv, c.round_bf16, c.synthetic_kv_seed = int(capture_kv), int(round_bf16), synthetic_kv_seed
    return c


class GenParams(C.Structure):
    _fields_ = [("n_requests", C.c_int), ("mean_interarrival", C.c_double),
                ("prompt_len_min", C.c_int), ("prompt_len_max", C.c_int),
                ("output_len_min", C.c_int), ("output_len_max", C.c_int),
                ("seed", C.c_uint64), ("vocab_size", C.c_int), ("eos_token", C.c_int)]


@dataclass
class Workload:
    arrival: np.ndarray
    prompt_off: np.ndarray
    prompt: np.ndarray
    max_new: np.ndarray

    @property
    def n(self) -> int:
        return len(self.arrival)

    @staticmethod
    def from_requests(reqs):
        """reqs: list of (arrival, [tokens], max_new)."""
        arrival = np.array([r[0] for r in reqs], dtype=np.float64)
        off = np.zeros(len(reqs) + 1, dtype=np.int32)
        toks = []
        for i, r in enumerate(reqs):
            toks.extend(r[1])
            off[i + 1] = len(toks)
        return Workload(arrival, off, np.array(toks, dtype=np.int32),
                        np.array([r[2] for r in reqs], dtype=np.int32))

    def prompts(self):
        return [self.prompt[self.prompt_off[i]:self.prompt_off[i + 1]].tolist() for i in range(self.n)]


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


@dataclass
class Transcript:
    """Flat transcript (same fields from port, reference and product)."""
    f: dict = field(default_factory=dict)

    def __getitem__(self, k):
        return self.f[k]

    @property
    def iterations(self):
        off = self.f["it_batch_off"]
        out = []
        for i in range(len(self.f["it_output_layer"])):
            a, b = off[i], off[i + 1]
            out.append(dict(clock=self.f["it_clock"][i], charge=self.f["it_charge"][i],
                            output_layer=int(self.f["it_output_layer"][i]),
                            batch_ids=self.f["ps_seq"][a:b].tolist(),
                            accept=self.f["ps_accept"][a:b].tolist(),
                            tokens=self.f["ps_token"][a:b].tolist()))
        return out

    @property
    def sequences(self):
        po, to = self.f["sq_prompt_off"], self.f["sq_tok_off"]
        out = []
        for i in range(len(self.f["sq_id"])):
            out.append(dict(id=int(self.f["sq_id"][i]), arrival=self.f["sq_arrival"][i],
                            first_token=self.f["sq_first"][i], finish=self.f["sq_finish"][i],
                            max_new=int(self.f["sq_max_new"][i]),
                            prompt=self.f["sq_prompt"][po[i]:po[i + 1]].tolist(),
                            tokens=self.f["sq_tokens"][to[i]:to[i + 1]].tolist(),
                            exit_layers=self.f["sq_exit_layers"][to[i]:to[i + 1]].tolist(),
                            iter_output_layers=self.f["sq_iter_out"][to[i]:to[i + 1]].tolist()))
        return out

    @property
    def final_clock(self):
        return float(self.f["meta"][0])


def read_flat(lib, prefix, handle) -> Transcript:
    t = Transcript()
    ln = getattr(lib, prefix + "transcript_len")
    for name in I32_FIELDS:
        n = ln(handle, name.encode())
        a = np.zeros(max(n, 0), dtype=np.int32)
        if n > 0:
            getattr(lib, prefix + "transcript_get_i32")(handle, name.encode(), _p(a, C.c_int32))
        t.f[name] = a
    for name in F64_FIELDS:
        n = ln(handle, name.encode())
        a = np.zeros(max(n, 0), dtype=np.float64)
        if n > 0:
            getattr(lib, prefix + "transcript_get_f64")(handle, name.encode(), _p(a, C.c_double))
        t.f[name] = a
    return t


class _Lib:
    prefix = ""
    so = ""

    def __init__(self):
        if not os.path.exists(self.so):
            raise FileNotFoundError(f"{self.so} not built (run oracle/Makefile)")
        self.lib = C.CDLL(self.so)
        L = self.lib
        p = self.prefix
        g = lambda n: getattr(L, p + n)  # noqa: E731
        g("last_error").restype = C.c_char_p
        g("model_free").argtypes = [C.c_void_p]
        g("model_tensor").argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_int64]
        g("gen_workload").restype = C.c_int64
        g("gen_workload").argtypes = [C.POINTER(GenParams), C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        g("transcript_len").restype = C.c_int64
        g("transcript_len").argtypes = [C.c_void_p, C.c_char_p]
        g("transcript_get_i32").argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_int32)]
        g("transcript_get_f64").argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_double)]
        g("transcript_free").argtypes = [C.c_void_p]
        g("transcript_kv").argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.c_int64]
        g("transcript_exit_states").argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.c_int64]
        for n in ["softmax_response_confidence"]:
            g(n).restype = C.c_double
            g(n).argtypes = [C.POINTER(C.c_double), C.c_int]
        g("state_similarity_confidence").restype = C.c_double
        g("state_similarity_confidence").argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int]
        g("classifier_confidence").restype = C.c_double
        g("classifier_confidence").argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_double, C.c_int]
        g("threshold_at").restype = C.c_double
        g("threshold_at").argtypes = [C.c_double, C.c_double, C.c_double, C.c_int]
        g("status_trace").argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                      C.POINTER(C.c_int32)]
        g("kv_block_trace").argtypes = [C.c_int] * 4 + [C.POINTER(C.c_int32)] * 2 + [C.c_int, C.c_int,
                                                                                      C.POINTER(C.c_int32)]
        g("reference_decode").argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int, C.c_int, C.c_int,
                                          C.POINTER(C.c_int32)]
        g("replay_sequence").argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int, C.POINTER(C.c_int32),
                                         C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double), C.POINTER(C.c_double)]
        g("session_create").restype = C.c_void_p
        g("session_create").argtypes = [C.c_void_p, C.POINTER(EngineConfig), C.c_int, C.POINTER(C.c_int32),
                                        C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_int32)]
        g("session_free").argtypes = [C.c_void_p]
        g("session_kv").argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]
        self._setup()

    def _setup(self):
        pass

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def err(self):
        return self.fn("last_error")().decode()

    # ---- model ----
    def model(self, n_layers, d_model, vocab, seed, round_bf16=False, encoder_len=0, n_heads=1, encoder_layers=0):
        """encoder_len > 0: the T5-mode extension (cross-attention over synthetic
        encoder states) -- the C restatement only; the compiled reference has no
        encoder, so parity of that mode is not pinned by it.  n_heads > 1 (extension, not in
        the reference): self- and cross-attention split into heads of d_model / n_heads features."""
        if encoder_len:
            if self.prefix != "eo_":
                raise ValueError("the reference has no encoder / cross-attention (SPEC.md:13, 184)")
            h = self.fn("model_seeded_t5")(n_layers, d_model, vocab, C.c_uint64(seed), int(round_bf16),
                                           int(encoder_len))
        else:
            h = self.fn("model_seeded")(n_layers, d_model, vocab, C.c_uint64(seed), int(round_bf16))
        if not h:
            raise ValueError(self.err())
        m = Model(self, h, n_layers, d_model, vocab, seed)
        m.encoder_len = encoder_len
        m.n_heads = n_heads
        if n_heads != 1 and self.fn("model_set_heads")(C.c_void_p(h), int(n_heads)):
            raise ValueError(self.err())
        m.encoder_layers = encoder_layers
        if encoder_layers and self.fn("model_set_encoder_layers")(C.c_void_p(h), int(encoder_layers)):
            raise ValueError(self.err())
        return m

    def gen_workload(self, n_requests=8, mean_interarrival=0.0, prompt_len_min=1, prompt_len_max=8,
                     output_len_min=1, output_len_max=16, seed=0, vocab_size=256, eos_token=0) -> Workload:
        gp = GenParams(n_requests, mean_interarrival, prompt_len_min, prompt_len_max, output_len_min,
                       output_len_max, seed, vocab_size, eos_token)
        tot = self.fn("gen_workload")(C.byref(gp), None, None, None, None)
        if tot < 0:
            raise ValueError(self.err())
        w = Workload(np.zeros(n_requests), np.zeros(n_requests + 1, np.int32), np.zeros(tot, np.int32),
                     np.zeros(n_requests, np.int32))
        self.fn("gen_workload")(C.byref(gp), _p(w.arrival, C.c_double), _p(w.prompt_off, C.c_int32),
                                _p(w.prompt, C.c_int32), _p(w.max_new, C.c_int32))
        return w

    def _transcript(self, h) -> Transcript:
        t = read_flat(self.lib, self.prefix, h)
        t.handle = h
        t.lib = self
        return t

    def transcript_kv(self, t, seq, layer, d):
        n = 1 << 22
        k = np.zeros(n); v = np.zeros(n)
        c = self.fn("transcript_kv")(t.handle, seq, layer, _p(k, C.c_double), _p(v, C.c_double), n)
        if c < 0:
            raise ValueError(self.err())
        return k[: c * d].reshape(c, d), v[: c * d].reshape(c, d)

    def transcript_block_table(self, t, seq, n_layers):
        """block table [L][bpl] of a captured sequence at eviction (C port only)"""
        f = self.fn("transcript_block_table")
        f.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int32), C.c_int64]
        out = np.zeros(1 << 20, np.int32)
        n = f(t.handle, seq, _p(out, C.c_int32), out.size)
        if n < 0:
            raise ValueError(self.err())
        return out[: n_layers * n].reshape(n_layers, n)

    def transcript_exit_states(self, t, seq, d):
        n = 1 << 22
        o = np.zeros(n)
        c = self.fn("transcript_exit_states")(t.handle, seq, _p(o, C.c_double), n)
        if c < 0:
            raise ValueError(self.err())
        return o[: c * d].reshape(c, d)

    def write_transcript_jsonl(self, t, path):
        """the reference's own writer (oracle/_ref only)"""
        rc = self.fn("transcript_write_jsonl")(t.handle, path.encode())
        if rc:
            raise RuntimeError(self.err())

    def write_report(self, t, path, fmt, wall=0.0):
        """compute_metrics + write_report of the reference itself (oracle/_ref only)"""
        f = self.fn("transcript_write_report")
        f.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_double]
        rc = f(t.handle, path.encode(), fmt.encode(), wall)
        if rc:
            raise RuntimeError(self.err())

    def free_transcript(self, t):
        if getattr(t, "handle", None):
            self.fn("transcript_free")(t.handle)
            t.handle = None

    # ---- single functions ----
    def softmax_response(self, logits):
        a = np.ascontiguousarray(logits, dtype=np.float64)
        return self.fn("softmax_response_confidence")(_p(a, C.c_double), len(a))

    def state_similarity(self, u, v):
        a = np.ascontiguousarray(u, dtype=np.float64); b = np.ascontiguousarray(v, dtype=np.float64)
        return self.fn("state_similarity_confidence")(_p(a, C.c_double), _p(b, C.c_double), len(a))

    def classifier(self, h, w, b):
        a = np.ascontiguousarray(h, dtype=np.float64); ww = np.ascontiguousarray(w, dtype=np.float64)
        return self.fn("classifier_confidence")(_p(a, C.c_double), _p(ww, C.c_double), b, len(a))

    def threshold_at(self, l0, g, lmin, layer):
        return self.fn("threshold_at")(l0, g, lmin, layer)

    def status_trace(self, conf, lambdas):
        conf = np.ascontiguousarray(conf, dtype=np.float64)
        L, B = conf.shape
        lam = np.ascontiguousarray(lambdas, dtype=np.float64)
        fa = np.zeros(B, np.int32)
        out = self.fn("status_trace")(B, L, _p(conf, C.c_double), _p(lam, C.c_double), _p(fa, C.c_int32))
        return out, fa

    def kv_block_trace(self, n_layers, pool, cap, ops, caps, n_ids, bpl_max):
        ops = np.ascontiguousarray(ops, dtype=np.int32); caps = np.ascontiguousarray(caps, dtype=np.int32)
        tab = np.zeros((n_ids, n_layers, bpl_max), np.int32)
        nf = self.fn("kv_block_trace")(n_layers, pool, cap, len(ops), _p(ops, C.c_int32), _p(caps, C.c_int32),
                                       n_ids, bpl_max, _p(tab, C.c_int32))
        if nf < 0:
            raise RuntimeError(self.err())
        return tab, nf


class Model:
    def __init__(self, lib, h, L, d, V, seed):
        self.lib, self.h, self.L, self.d, self.V, self.seed = lib, h, L, d, V, seed

    def __del__(self):
        try:
            if self.h:
                self.lib.fn("model_free")(self.h)
        except Exception:
            pass

    def encoder_state(self, seq_id, t):
        out = np.zeros(self.d)
        self.lib.fn("encoder_state")(self.h, seq_id, t, _p(out, C.c_double))
        return out

    def encoder_token(self, seq_id, t):
        """seeded encoder input id of (sequence, position) (T5 encoder stack)"""
        f = self.lib.fn("encoder_token")
        f.argtypes = [C.c_void_p, C.c_int, C.c_int]
        return int(f(self.h, seq_id, t))

    def tensor(self, which, layer=0):
        names = {"embedding": 0, "lm_head": 1, "probe_w": 2, "probe_b": 3, "w_q": 4, "w_k": 5, "w_v": 6,
                 "w_o": 7, "w_up": 8, "w_down": 9, "w_qc": 10, "w_kc": 11, "w_vc": 12, "w_oc": 13,
                 "e_q": 20, "e_k": 21, "e_v": 22, "e_o": 23, "e_up": 24, "e_down": 25}
        w = names[which] if isinstance(which, str) else which
        d, V = self.d, self.V
        shape = {0: (V, d), 1: (V, d), 2: (d,), 3: (1,), 4: (d, d), 5: (d, d), 6: (d, d), 7: (d, d),
                 8: (4 * d, d), 9: (d, 4 * d), 10: (d, d), 11: (d, d), 12: (d, d), 13: (d, d),
                 20: (d, d), 21: (d, d), 22: (d, d), 23: (d, d), 24: (4 * d, d), 25: (d, 4 * d)}[w]
        out = np.zeros(int(np.prod(shape)))
        rc = self.lib.fn("model_tensor")(self.h, w, layer, _p(out, C.c_double), out.size)
        if rc:
            raise ValueError(self.lib.err())
        return out.reshape(shape)

    def run(self, cfg: EngineConfig, wl: Workload, fixed_conf=None) -> Transcript:
        return self.lib.engine_run(self, cfg, wl, fixed_conf)

    def reference_decode(self, prompt, max_new, eos):
        p = np.ascontiguousarray(prompt, dtype=np.int32)
        out = np.zeros(max_new, np.int32)
        n = self.lib.fn("reference_decode")(self.h, _p(p, C.c_int32), len(p), max_new, eos, _p(out, C.c_int32))
        if n < 0:
            raise ValueError(self.lib.err())
        return out[:n].tolist()

    def replay_sequence(self, prompt, exits):
        p = np.ascontiguousarray(prompt, dtype=np.int32)
        e = np.ascontiguousarray(exits, dtype=np.int32)
        n, d, L = len(e), self.d, self.L
        P = len(p) - 1 + n
        toks = np.zeros(n, np.int32)
        hs = np.zeros((n, d))
        kk = np.zeros((L, P, d)); vv = np.zeros((L, P, d))
        rc = self.lib.fn("replay_sequence")(self.h, _p(p, C.c_int32), len(p), _p(e, C.c_int32), n,
                                            _p(toks, C.c_int32), _p(hs, C.c_double), _p(kk, C.c_double),
                                            _p(vv, C.c_double))
        if rc:
            raise ValueError(self.lib.err())
        return dict(tokens=toks.tolist(), exit_states=hs, k=kk, v=vv)

    def session(self, cfg, first_tokens, prefix_len, capacity, kv_seed, seq_ids=None):
        return Session(self, cfg, first_tokens, prefix_len, capacity, kv_seed, seq_ids)


class Session:
    """Fixed batch decode over a seeded KV prefix (restated decode_iteration)."""

    def __init__(self, model, cfg, first_tokens, prefix_len, capacity, kv_seed, seq_ids=None):
        self.m = model
        self.cfg = cfg
        ft = np.ascontiguousarray(first_tokens, dtype=np.int32)
        self.B = len(ft)
        ids = np.ascontiguousarray(seq_ids if seq_ids is not None else np.arange(self.B), dtype=np.int32)
        self.h = model.lib.fn("session_create")(model.h, C.byref(cfg), self.B, _p(ft, C.c_int32), prefix_len,
                                                capacity, C.c_uint64(kv_seed), _p(ids, C.c_int32))
        if not self.h:
            raise ValueError(model.lib.err())

    def __del__(self):
        try:
            if self.h:
                self.m.lib.fn("session_free")(self.h)
        except Exception:
            pass

    def step(self, forced=0, fixed_conf=None, tokens_in=None):
        """One decode iteration. forced>0 replays a recorded output layer;
        tokens_in overrides the inputs (teacher forcing from another engine)."""
        B, L, d = self.B, self.m.L, self.m.d
        toks = np.zeros(B, np.int32); acc = np.zeros(B, np.int32)
        conf = np.zeros((L, B)); hx = np.zeros((B, d))
        tin = np.ascontiguousarray(tokens_in, dtype=np.int32) if tokens_in is not None else None
        lib = self.m.lib
        if lib.prefix == "eo_":
            fc = np.ascontiguousarray(fixed_conf, dtype=np.float64) if fixed_conf is not None else None
            e = lib.fn("session_step")(self.h, forced, _p(fc, C.c_double), _p(tin, C.c_int32), _p(toks, C.c_int32),
                                       _p(acc, C.c_int32), _p(conf, C.c_double), _p(hx, C.c_double))
        else:
            if fixed_conf is not None:
                raise ValueError("the reference session has no injected-confidence mode")
            e = lib.fn("session_step")(self.h, forced, _p(tin, C.c_int32), _p(toks, C.c_int32), _p(acc, C.c_int32),
                                       _p(conf, C.c_double), _p(hx, C.c_double))
        if e < 0:
            raise RuntimeError(lib.err())
        return dict(output_layer=e, tokens=toks, accept=acc, conf=conf, h_exit=hx)

    def set_per_seq_exit(self, on=True):
        """layer-level scheduling semantics: each row exits at its own first accept (C port only)"""
        if self.m.lib.fn("session_set_per_seq_exit")(self.h, int(on)):
            raise ValueError(self.m.lib.err())

    # layer-stepped iteration (reference only): a batch sharded over processes keeps the
    # reference's batch-wide exit barrier (oracle/ref_capi.cpp ref_session_iter_*)
    def iter_begin(self, tokens_in=None):
        tin = np.ascontiguousarray(tokens_in, dtype=np.int32) if tokens_in is not None else None
        if self.m.lib.fn("session_iter_begin")(self.h, _p(tin, C.c_int32)):
            raise RuntimeError(self.m.lib.err())

    def iter_layer(self, layer) -> bool:
        r = self.m.lib.fn("session_iter_layer")(self.h, layer)
        if r < 0:
            raise RuntimeError(self.m.lib.err())
        return bool(r)

    def iter_finish(self, output_layer):
        toks = np.zeros(self.B, np.int32); acc = np.zeros(self.B, np.int32)
        if self.m.lib.fn("session_iter_finish")(self.h, output_layer, _p(toks, C.c_int32), _p(acc, C.c_int32)):
            raise RuntimeError(self.m.lib.err())
        return toks, acc

    def kv(self, row, layer, pos):
        d = self.m.d
        k = np.zeros(d); v = np.zeros(d)
        rc = self.m.lib.fn("session_kv")(self.h, row, layer, pos, _p(k, C.c_double), _p(v, C.c_double))
        if rc:
            raise ValueError(self.m.lib.err())
        return k, v


class Port(_Lib):
    prefix = "eo_"
    so = PORT_SO

    def _setup(self):
        L = self.lib
        L.eo_model_seeded.restype = C.c_void_p
        L.eo_model_seeded.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int]
        L.eo_model_seeded_t5.restype = C.c_void_p
        L.eo_model_seeded_t5.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int]
        L.eo_encoder_state.restype = None
        L.eo_encoder_state.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.eo_engine_run.argtypes = [C.c_void_p, C.POINTER(EngineConfig), C.c_int, C.POINTER(C.c_double),
                                    C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_void_p)]
        L.eo_session_step.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double)]
        # (a handle passed without argtypes would be truncated to a C int)
        L.eo_session_set_per_seq_exit.argtypes = [C.c_void_p, C.c_int]
        L.eo_round_bf16.restype = C.c_double
        L.eo_round_bf16.argtypes = [C.c_double]
        L.eo_splitmix64_at.restype = C.c_uint64
        L.eo_splitmix64_at.argtypes = [C.c_uint64, C.c_uint64]
        L.eo_kv_prefix_vector.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_int, C.POINTER(C.c_double)]

    def engine_run(self, model, cfg, wl: Workload, fixed_conf=None) -> Transcript:
        h = C.c_void_p()
        nfix = 0
        fc = None
        if fixed_conf is not None:
            fc = np.ascontiguousarray(fixed_conf, dtype=np.float64)
            nfix = fc.shape[0]
        rc = self.lib.eo_engine_run(model.h, C.byref(cfg), wl.n, _p(wl.arrival, C.c_double),
                                    _p(wl.prompt_off, C.c_int32), _p(wl.prompt, C.c_int32),
                                    _p(wl.max_new, C.c_int32), _p(fc, C.c_double), nfix, C.byref(h))
        if rc:
            raise RuntimeError(f"eo_engine_run rc={rc}: {self.err()}")
        return self._transcript(h)

    def kv_prefix_vector(self, kv_seed, L, seq, layer, pos, kind, d, rb=True):
        out = np.zeros(d)
        self.lib.eo_kv_prefix_vector(kv_seed, L, seq, layer, pos, kind, d, int(rb), _p(out, C.c_double))
        return out


class Ref(_Lib):
    prefix = "ref_"
    so = REF_SO

    def _setup(self):
        L = self.lib
        L.ref_model_seeded.restype = C.c_void_p
        L.ref_model_seeded.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int]
        L.ref_engine_run.argtypes = [C.c_void_p, C.POINTER(EngineConfig), C.c_int, C.POINTER(C.c_double),
                                     C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                     C.POINTER(C.c_void_p)]
        L.ref_session_step.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_greedy_token.argtypes = [C.POINTER(C.c_double), C.c_int]
        L.ref_session_iter_begin.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
        L.ref_session_iter_layer.argtypes = [C.c_void_p, C.c_int]
        L.ref_session_iter_finish.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]

    def engine_run(self, model, cfg, wl: Workload, fixed_conf=None) -> Transcript:
        if fixed_conf is not None:
            raise ValueError("the reference engine has no injected-confidence mode")
        h = C.c_void_p()
        rc = self.lib.ref_engine_run(model.h, C.byref(cfg), wl.n, _p(wl.arrival, C.c_double),
                                     _p(wl.prompt_off, C.c_int32), _p(wl.prompt, C.c_int32),
                                     _p(wl.max_new, C.c_int32), C.byref(h))
        if rc:
            raise RuntimeError(f"ref_engine_run rc={rc}: {self.err()}")
        return self._transcript(h)


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def ref() -> Ref | None:
    """The compiled reference, or None where it was never built (GPU box without _ref)."""
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        _ref = Ref()
    return _ref
