"""Qwen3-32B-shaped stack driver of TN projections (BASELINE cfg4).

64 decoder layers x {q 5120->8192, k/v 5120->1024, o 8192->5120, gate/up 5120->25600,
down 25600->5120}, all TN-compressed with the pinned "sensitivity-mix" layout of SURVEY §8(d):
  q/o Tucker-2 R256; k/v Tucker-2 R128;
  MLP: layers 0-1 and 62-63 Tucker-2 R256 (fragile edges, mirroring planner.py:140-143);
       other layers rotate by l mod 3 among TT r64, TR4 (4,16,16,16) and
       Tucker-4 (32,32,16,16) (down: (16,16,32,32)).
Mode shapes come from ``default_mode_shape`` (tn_decompositions.py:59-63); Tucker-2 uses the
two-mode (rows | cols) shape.

The attention core is not part of the TN-linear path: it is a pass-through (the attention
output is taken to be q). Pre-norm as in Qwen3 (RMSNorm without learned scale), per layer:
  h = rms(x); q, k, v = Lq(h), Lk(h), Lv(h);  x = x + Lo(q)
  h = rms(x); x = x + Ld(silu(Lg(h)) * Lu(h))
The projections run through libtnl (tnl_forward); the MLP half runs as one ``TNMLP`` block
(tnl_mlp_forward: gate/up/SiLU*mul/down fused with h on chip for prefill-sized M and
merged-cut ranks <= 128, the dual gate/up kernel for larger ranks, else three layers around a
SiLU*mul kernel); each residual add is fused with the next RMSNorm into one pass
(``tnl_add_rmsnorm``: x += o; h = rms(x)). All plans and MLP blocks share one workspace.
``capture(m)`` records one whole pass into a CUDA graph.
"""

from __future__ import annotations

import ctypes
import time

import torch

from . import _native as N
from .errors import UnsupportedError
from . import synthetic as S
from .mlp import TNMLP
from .stack import TNGroup
from .modes import default_mode_shape

HIDDEN, QDIM, KVDIM, FFN = 5120, 8192, 1024, 25600


def _tn(kind: str, rows: int, cols: int, seed: int):
    if kind.startswith("tucker2-"):
        r = int(kind.split("-")[1])
        return S.make_layer("tucker", (rows, cols), 1, (r, r), seed)
    ms, rm = default_mode_shape(rows, cols)
    if kind == "tt64":
        return S.make_layer("tt", ms, rm, (64,) * (len(ms) - 1), seed)
    if kind == "tr4":
        return S.make_layer("tr", ms, rm, (4, 16, 16, 16), seed)
    if kind == "tucker4":
        ranks = (32, 32, 16, 16) if rows > cols else (16, 16, 32, 32)
        return S.make_layer("tucker", ms, rm, ranks, seed)
    raise ValueError(kind)


def layer_kinds(l: int, n_layers: int = 64) -> dict:
    mlp = "tucker2-256" if (l < 2 or l >= n_layers - 2) else ("tt64", "tr4", "tucker4")[l % 3]
    return {"q": "tucker2-256", "k": "tucker2-128", "v": "tucker2-128", "o": "tucker2-256",
            "gate": mlp, "up": mlp, "down": mlp}


SHAPES = {"q": (QDIM, HIDDEN), "k": (KVDIM, HIDDEN), "v": (KVDIM, HIDDEN), "o": (HIDDEN, QDIM),
          "gate": (FFN, HIDDEN), "up": (FFN, HIDDEN), "down": (HIDDEN, FFN)}


class QwenTNStack:
    def __init__(self, n_layers: int = 64, dtype=torch.bfloat16, device=None, seed: int = 40_000,
                 fused_mlp: bool = True, mlp_kinds=None):
        """mlp_kinds: optional per-layer MLP family override (e.g. ["tt64", "tr4", "tucker4"]) so
        short stacks can exercise every cfg4 layer variant; default: the sensitivity-mix layout."""
        self.n_layers = n_layers
        self.dtype = dtype
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.layers = []
        self.build_s = {"host_cores": 0.0, "device_plans": 0.0}  # construction time split
        for l in range(n_layers):
            kinds = layer_kinds(l, n_layers)
            if mlp_kinds is not None:
                kinds.update(gate=mlp_kinds[l], up=mlp_kinds[l], down=mlp_kinds[l])
            blk = {}
            for j, name in enumerate(("q", "k", "v", "o", "gate", "up", "down")):
                rows, cols = SHAPES[name]
                t0 = time.perf_counter()
                layer = _tn(kinds[name], rows, cols, seed=seed + 100 * l + 10 * j)
                t1 = time.perf_counter()
                blk[name] = (kinds[name], layer, layer.plan(dtype, self.device))
                self.build_s["host_cores"] += t1 - t0
                self.build_s["device_plans"] += time.perf_counter() - t1
            t1 = time.perf_counter()
            blk["mlp"] = TNMLP(blk["gate"][1], blk["up"][1], blk["down"][1], dtype=dtype, device=self.device,
                               fused=fused_mlp)
            # prefill: k, v and q read the same normalised hidden state -> one stacked first step
            blk["kvq"] = TNGroup([blk["k"][1], blk["v"][1], blk["q"][1]], dtype=dtype, device=self.device)
            self.build_s["device_plans"] += time.perf_counter() - t1
            # decode: q -> (pass-through attention) -> o as one two-layer stack (one fused
            # boundary kernel: q's output rows never leave the SM)
            blk["qo"] = (ctypes.c_void_p * 2)(blk["q"][2].handle.value, blk["o"][2].handle.value)
            self.layers.append(blk)
        self.fuse_qo = True
        # prefill: residual adds and RMSNorms folded into the projections' epilogues (tnl_fwd_opts)
        self.fold_prefill = True
        self.group_kvq = True
        self.fuse_rms = True  # RMS statistics summed inside the stacked input steps
        self._ws = None
        self._ws_side = None
        self._side = None
        # decode: k and v (independent of q given h) run on a forked stream with their own workspace
        self.concurrent_kv = True

    def param_count(self) -> int:
        from .layer import param_count

        return sum(param_count(lay) for _, lay, _ in self.projections())

    def projections(self):
        return [blk[n] for blk in self.layers for n in ("q", "k", "v", "o", "gate", "up", "down")]

    def chain_flops_per_token(self) -> int:
        return sum(lay.chain_flops_per_token() for _, lay, _ in self.projections())

    def fused_mlp_count(self) -> int:
        return sum(blk["mlp"].fused for blk in self.layers)

    def workspace(self, m: int):
        need = max(max(p.workspace_bytes(m) for _, _, p in self.projections()),
                   max(blk["mlp"].workspace_bytes(m) for blk in self.layers),
                   max(blk["kvq"].workspace_bytes(m) for blk in self.layers))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(max(need, 256), dtype=torch.uint8, device=self.device)
        return self._ws

    def _side_workspace(self, m: int):
        need = max(max(blk[n][2].workspace_bytes(m) for n in ("k", "v")) for blk in self.layers)
        if self._ws_side is None or self._ws_side[0].numel() < need:
            self._ws_side = [torch.zeros(max(need, 256), dtype=torch.uint8, device=self.device) for _ in range(2)]
        if self._side is None:
            self._side = [torch.cuda.Stream(self.device) for _ in range(2)]
        return self._ws_side

    def _group_ctx(self, m: int):
        """Private workspaces (zero-filled: decode accumulators) and k/v side streams for one
        concurrently running token group (decode microbatches)."""
        need = max(max(p.workspace_bytes(m) for _, _, p in self.projections()),
                   max(blk["mlp"].workspace_bytes(m) for blk in self.layers),
                   max(blk["kvq"].workspace_bytes(m) for blk in self.layers))
        need_side = max(max(blk[n][2].workspace_bytes(m) for n in ("k", "v")) for blk in self.layers)
        z = lambda n: torch.zeros(max(n, 256), dtype=torch.uint8, device=self.device)  # noqa: E731
        return {"ws": z(need), "ws_side": [z(need_side), z(need_side)],
                "side": [torch.cuda.Stream(self.device) for _ in range(2)]}

    def _buffers(self, m: int):
        mk = lambda n: torch.empty((m, n), dtype=self.dtype, device=self.device)  # noqa: E731
        return {"h": mk(HIDDEN), "q": mk(QDIM), "k": mk(KVDIM), "v": mk(KVDIM), "o": mk(HIDDEN), "d": mk(HIDDEN),
                "ss": torch.zeros((2, m), dtype=torch.float32, device=self.device)}

    @staticmethod
    def add_rmsnorm(x: torch.Tensor, o, h: torch.Tensor, eps: float = 1e-6) -> None:
        """x += o (if o is not None); h = x / rms(x) — one pass (tnl_add_rmsnorm)."""
        m, n = x.shape
        stream = torch.cuda.current_stream(x.device).cuda_stream
        optr = ctypes.c_void_p(o.data_ptr()) if o is not None else None
        N.check(N.load().tnl_add_rmsnorm(ctypes.c_void_p(x.data_ptr()), x.stride(0), optr,
                                         o.stride(0) if o is not None else 0, ctypes.c_void_p(h.data_ptr()),
                                         h.stride(0), m, n, float(eps), ctypes.c_void_p(stream)))

    def _forward_prefill_folded(self, x: torch.Tensor, b, ws) -> torch.Tensor:
        """Prefill pass with the residual adds and RMSNorms folded into the TN kernels
        (tnl_fwd_opts): per norm one statistics read of x (tnl_rms_stats) replaces the add+norm pass;
        q/k/v and gate/up scale their cut activations by 1/rms(x); o and the MLP add their output
        into x with the TMA store's reduce-add (residual stream updated in place)."""
        lib = N.load()
        m = x.shape[0]
        st = ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        ss = b["ss"][0]
        eps = 1e-6
        o_norm = N.FwdOpts(0, ss.data_ptr(), HIDDEN, eps)
        o_acc = N.FwdOpts(1, None, 0, 0.0)
        o_both = N.FwdOpts(1, ss.data_ptr(), HIDDEN, eps)
        # rms_fused: the stacked k/v/q and gate/up input steps sum the squares of x themselves while
        # streaming it (no statistics pass over x); on TNL_ERR_UNSUPPORTED (a K-split step) the
        # statistics pass + ss_in is used instead
        o_norm_f = N.FwdOpts(0, None, HIDDEN, eps, 1)
        o_both_f = N.FwdOpts(1, None, HIDDEN, eps, 1)

        def fused_or_stats(run_fused, run_stats):
            if self.fuse_rms and self.group_kvq:
                try:
                    run_fused()
                    return
                except UnsupportedError:
                    pass
            N.check(lib.tnl_rms_stats(vp(x), x.stride(0), m, HIDDEN, vp(ss), st))
            run_stats()

        for blk in self.layers:
            if self.group_kvq:  # one first step over x for k, v and q (x read once)
                fused_or_stats(lambda: blk["kvq"].forward(x, outs=[b["k"], b["v"], b["q"]], ws=ws, opts=o_norm_f),
                               lambda: blk["kvq"].forward(x, outs=[b["k"], b["v"], b["q"]], ws=ws, opts=o_norm))
            else:
                N.check(lib.tnl_rms_stats(vp(x), x.stride(0), m, HIDDEN, vp(ss), st))
                for name in ("k", "v", "q"):
                    pl = blk[name][2]
                    N.check(lib.tnl_forward_ex(pl.handle, vp(x), m, x.stride(0), vp(b[name]), b[name].stride(0),
                                               vp(ws), ws.numel(), ctypes.byref(o_norm), st))
            pl = blk["o"][2]  # attention core: pass-through; x += o
            N.check(lib.tnl_forward_ex(pl.handle, vp(b["q"]), m, b["q"].stride(0), vp(x), x.stride(0), vp(ws),
                                       ws.numel(), ctypes.byref(o_acc), st))
            fused_or_stats(  # x += mlp(norm(x))
                lambda: N.check(lib.tnl_mlp_forward_ex(blk["mlp"].handle, vp(x), m, x.stride(0), vp(x), x.stride(0),
                                                       vp(ws), ws.numel(), ctypes.byref(o_both_f), st)),
                lambda: N.check(lib.tnl_mlp_forward_ex(blk["mlp"].handle, vp(x), m, x.stride(0), vp(x), x.stride(0),
                                                       vp(ws), ws.numel(), ctypes.byref(o_both), st)))
        return x

    def forward(self, x: torch.Tensor, bufs=None, ctx=None) -> torch.Tensor:
        """One pass of all layers; x (M x 5120) is updated in place (residual stream). `ctx`
        (from _group_ctx) gives a token group its own workspaces and side streams."""
        m = x.shape[0]
        ws = ctx["ws"] if ctx else self.workspace(m)
        b = bufs or self._buffers(m)
        if self.fold_prefill and m > 64:
            if "ss" not in b:
                b["ss"] = torch.zeros((2, m), dtype=torch.float32, device=self.device)
            return self._forward_prefill_folded(x, b, ws)
        fork = self.concurrent_kv and m <= 64
        side = self._side
        if fork:
            if ctx:
                ws_side, side = ctx["ws_side"], ctx["side"]
            else:
                ws_side = self._side_workspace(m)
                side = self._side
            cur = torch.cuda.current_stream(self.device)
        for li, blk in enumerate(self.layers):
            # x += previous MLP output; h = rms(x)   (fused residual add + RMSNorm, one pass)
            self.add_rmsnorm(x, b["d"] if li else None, b["h"])
            if fork:
                # k and v on two forked streams (own zero-at-rest workspaces): each is two kernels,
                # shorter than the q -> o chain, so neither is on the critical path; joined before h is
                # overwritten
                for j, name in enumerate(("k", "v")):
                    side[j].wait_stream(cur)
                    with torch.cuda.stream(side[j]):
                        blk[name][2].forward(b["h"], out=b[name], ws=ws_side[j])
            else:
                blk["k"][2].forward(b["h"], out=b["k"], ws=ws)
                blk["v"][2].forward(b["h"], out=b["v"], ws=ws)
            if fork and self.fuse_qo:
                st = torch.cuda.current_stream(self.device).cuda_stream
                N.check(N.load().tnl_stack_forward(blk["qo"], 2, ctypes.c_void_p(b["h"].data_ptr()), m,
                                                   b["h"].stride(0) if m > 1 else HIDDEN,
                                                   ctypes.c_void_p(b["o"].data_ptr()),
                                                   b["o"].stride(0) if m > 1 else HIDDEN,
                                                   ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.c_void_p(st)))
            else:
                blk["q"][2].forward(b["h"], out=b["q"], ws=ws)
                blk["o"][2].forward(b["q"], out=b["o"], ws=ws)  # attention core: pass-through
            if fork:
                for sd in side:
                    cur.wait_stream(sd)
            self.add_rmsnorm(x, b["o"], b["h"])
            blk["mlp"].forward(b["h"], out=b["d"], ws=ws)
        x.add_(b["d"])
        return x

    def capture(self, m: int, microbatches: int = 1):
        """Record one pass for M = m tokens into a CUDA graph. Decode (m <= 64) may split the
        tokens into `microbatches` groups that run the whole stack concurrently on forked streams,
        each with its own workspaces (tokens are independent through the stack: the attention core
        is a pass-through)."""
        self.x = torch.zeros((m, HIDDEN), dtype=self.dtype, device=self.device)
        k = max(1, min(microbatches, m)) if m <= 64 else 1
        bounds = [(i * m // k, (i + 1) * m // k) for i in range(k)]
        if k == 1:
            self.bufs = self._buffers(m)
            self.workspace(m)
            groups = [(0, m, self.bufs, None)]
        else:
            groups = [(lo, hi, self._buffers(hi - lo), self._group_ctx(hi - lo)) for lo, hi in bounds]
            self.bufs = groups[0][2]
        gstreams = [torch.cuda.Stream(self.device) for _ in groups]
        s = torch.cuda.Stream(self.device)

        def one_pass():
            fork = torch.cuda.Event()
            fork.record(s)
            joins = []
            for (lo, hi, bufs, ctx), gs in zip(groups, gstreams):
                gs.wait_event(fork)
                with torch.cuda.stream(gs):
                    self.forward(self.x[lo:hi], bufs, ctx)
                    e = torch.cuda.Event()
                    e.record(gs)
                    joins.append(e)
            for e in joins:
                s.wait_event(e)

        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            one_pass()
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            one_pass()
        self.graph = g
        self.microbatches = k
        return g
