"""Captured online-answer plans: fixed device buffers + CUDA graphs.

One plan per (state, thread, key width, output stride). Its input buffers
(qu, cko) and output (t) have fixed addresses, so the whole device sequence
-- query planes, compression operand, the two tcgen05 GEMMs, the group
stage -- is captured once into CUDA graphs and replayed per query:

  full graph     GEMV on (SMs - COMPRESS_CTAS) SMs || compression + the
                 Montgomery group stage (tz = Z_g mod m) on a side stream on
                 COMPRESS_CTAS SMs, joined by the finish (t = tz + B_g mod m)
                 (device-resident throughput; bench `value`)
  gemv graph     query planes + GEMV on all SMs
  compress graph compression operand + compression GEMM (all SMs) + groups
                 (respond(): the host converts ck_o while the gemv graph runs)

The eager sequence is run once before capture (sets kernel attributes,
warms the TMA-descriptor path).
"""

import threading

import numpy as np
import torch

from . import _lib, device

USE_GRAPHS = True     # False runs the sequences eagerly (debugging)
_capture_lock = threading.Lock()
# SMs the host-input graphs add to the compression side (it starts ~25 us after
# the GEMV: ck_o is staged while the GEMV runs)
E2E_EXTRA_CTAS = 8


class AnswerPlan:
    def __init__(self, state, kctx, t_ld, compress_ctas):
        lay = state.layout
        dev = state.device
        lm = kctx.lm
        if lm not in device.UMMA_NB or lay.qmask != 0xFFFFFFFF or state.engine != "umma":
            raise NotImplementedError("plans cover the tcgen05 path (lm 32/64/96, q = 2^32)")
        self.state, self.kctx, self.t_ld = state, kctx, t_ld
        self.ctas = compress_ctas
        # the host-input graphs start the compression side ~25 us after the
        # GEMV (ck_o is staged while the GEMV runs), so they give it more SMs
        self.ctas_e2e = compress_ctas + E2E_EXTRA_CTAS if compress_ctas > 0 else 0
        self.sms = torch.cuda.get_device_properties(dev).multi_processor_count
        self.qu = torch.zeros((1, lay.ld), dtype=torch.int32, device=dev)
        self.cko = torch.zeros((lay.n, lm), dtype=torch.int32, device=dev)
        self.planes = torch.empty((16, lay.ld), dtype=torch.uint8, device=dev)
        self.b = torch.empty((1, lay.rows), dtype=torch.int32, device=dev)
        self.bc = torch.empty(state.compress_operand_shape(lm), dtype=torch.uint8, device=dev)
        self.z = torch.empty((lay.rows, lm + 4), dtype=torch.int32, device=dev)
        self.t = torch.empty((lay.groups, t_ld), dtype=torch.int32, device=dev)
        self.tz = torch.empty((lay.groups, t_ld), dtype=torch.int32, device=dev)
        # pinned host mirrors for respond(): written in place, copied async
        self.h_qu = torch.zeros((lay.ld,), dtype=torch.int32).pin_memory()
        self.h_cko = torch.empty((lay.n, lm), dtype=torch.int32).pin_memory()
        self.h_t = torch.empty((lay.groups, t_ld), dtype=torch.int32).pin_memory()
        self.h_K = torch.empty((lay.groups, kctx.l2), dtype=torch.int32).pin_memory()
        # raw CPython 30-bit digits at the API boundary (regrouped on the device)
        self.ndig_m = -(-32 * lm // 30)
        self.ndig_2 = -(-32 * kctx.l2 // 30)
        self.d_ckd = torch.zeros((lay.n, self.ndig_m), dtype=torch.int32, device=dev)
        self.h_ckd = torch.zeros((lay.n, self.ndig_m), dtype=torch.int32).pin_memory()
        self.d_td = torch.zeros((lay.groups, self.ndig_m), dtype=torch.int32, device=dev)
        self.h_td = torch.zeros((lay.groups, self.ndig_m), dtype=torch.int32).pin_memory()
        self.d_Kd = torch.zeros((lay.groups, self.ndig_2), dtype=torch.int32, device=dev)
        self.h_Kd = torch.zeros((lay.groups, self.ndig_2), dtype=torch.int32).pin_memory()
        # numpy views of the pinned buffers (made once: respond() is latency-bound)
        self.np_qu = self.h_qu.numpy().view(np.uint32)
        self.np_ckd = self.h_ckd.numpy()
        self.np_td = self.h_td.numpy()
        self.np_Kd = self.h_Kd.numpy()
        # the client's modulus constants live in plan buffers read by the
        # captured group stage (refreshed by set_key when the client changes)
        self.nchunks = max(2, -(-(lay.cap + lm + 4) // lm))
        self.d_m = torch.zeros((1, lm), dtype=torch.int32, device=dev)
        self.d_rpow = torch.zeros((1, self.nchunks, lm), dtype=torch.int32, device=dev)
        self.d_np = torch.zeros((1,), dtype=torch.int32, device=dev)
        self.d_f0 = torch.zeros((1,), dtype=torch.uint8, device=dev)
        self.key_m = None
        self.side = torch.cuda.Stream(dev)
        self.ev_in = torch.cuda.Event()
        self.ev_comp = torch.cuda.Event()
        self.graphs = {}
        self.gemv_events = (torch.cuda.Event(enable_timing=True),
                            torch.cuda.Event(enable_timing=True))
        self.side_events = (torch.cuda.Event(enable_timing=True),
                            torch.cuda.Event(enable_timing=True))
        for e in self.gemv_events + self.side_events:   # torch creates the cudaEvent_t on first record
            e.record(torch.cuda.current_stream(dev))
        # respond(): the GEMV graph's completion, recorded outside the graphs
        self.ev_gemv = torch.cuda.Event()
        self.ev_gemv.record(torch.cuda.current_stream(dev))
        self._exec = {}
        # respond()'s host-input graphs read qu / ck_o's digits from and write
        # t's digits to the pinned host buffers directly (no copy nodes) when
        # the device address of each is its host address (UVA); else copies
        self.zero_copy = all(_mapped_in_place(b) for b in (self.h_qu, self.h_ckd, self.h_td))

    # -- eager pieces (also what gets captured) -----------------------------

    def _gemv(self, stream, ctas):
        device.query_planes(self.qu, 16, stream, planes=self.planes)
        device.umma_gemv(self.state.dbt, self.planes, 1, out=self.b, stream=stream, ctas=ctas)

    def _compress(self, stream, ctas):
        self.state.compress_rows(self.cko, self.kctx.lm, stream, out=self.z, ctas=ctas, bc=self.bc)

    def set_key(self, kctx, stream):
        """Load a client's modulus constants into the plan buffers (in-stream);
        True when they changed."""
        if self.key_m == kctx.m:
            return False
        import numpy as np
        with torch.cuda.stream(stream):
            self.d_m[0].copy_(kctx.d_m)
            self.d_rpow[0].copy_(kctx.d_rpow(self.nchunks))
            self.d_np.copy_(torch.tensor(np.array([kctx.cm.np], np.uint32).view(np.int32)),
                            non_blocking=False)
            self.d_f0.fill_(1 if kctx.cm.R < 2 * kctx.m else 0)
        self.kctx = kctx
        self.key_m = kctx.m
        return True

    def _groups_z(self, stream):
        """Montgomery part of the group stage; needs only the compression."""
        lay = self.state.layout
        device.groups_z(self.z, lay.d1, lay.cap, lay.groups, self.kctx.lm, self.d_m, self.d_np,
                        self.d_rpow, self.nchunks, self.d_f0, self.tz, self.t_ld, stream)

    def _finish(self, stream):
        """t = (tz + B) mod m once the GEMV's b is complete."""
        lay = self.state.layout
        device.groups_finish(self.tz, self.b, lay.qmask, lay.d1, lay.cap, lay.groups,
                             self.kctx.lm, self.d_m, self.t, self.t_ld, stream)

    def _seq(self, which, stream):
        if which in ("full", "full_timed"):
            # full_timed: the same step with timing events around the GEMV
            # (query planes + GEMV) on the main stream, for the in-step roofline
            tev = self.gemv_events if which == "full_timed" else None
            if self.ctas > 0:
                self.ev_in.record(stream)
                self.side.wait_event(self.ev_in)
                if tev:
                    device.event_record(self.side_events[0], self.side)
                self._compress(self.side, self.ctas)
                self._groups_z(self.side)      # overlaps the GEMV's tail
                if tev:
                    device.event_record(self.side_events[1], self.side)
                self.ev_comp.record(self.side)
                if tev:
                    device.event_record(tev[0], stream)
                self._gemv(stream, self.sms - self.ctas)
                if tev:
                    device.event_record(tev[1], stream)
                stream.wait_event(self.ev_comp)
            else:
                if tev:
                    device.event_record(tev[0], stream)
                self._gemv(stream, 0)
                if tev:
                    device.event_record(tev[1], stream)
                self._compress(stream, 0)
                self._groups_z(stream)
            self._finish(stream)
        elif which == "gemv":
            self._gemv(stream, 0)
        elif which == "compress":
            self._compress(stream, 0)
            self._groups_z(stream)
            self._finish(stream)
        elif which == "gemv_part":
            # respond(): GEMV on the SMs the side stream does not take
            self._gemv(stream, self.sms - self.ctas if self.ctas > 0 else 0)
        elif which == "side_digits":
            # respond(), side stream: ck_o digits -> limbs, compression, Montgomery groups
            device.digits_to_limbs(self.d_ckd, self.kctx.lm, self.cko, stream)
            self._compress(stream, self.ctas)
            self._groups_z(stream)
        elif which == "e2e_digits":
            # respond() in one replay: both host->device copies, GEMV || (ck_o
            # digits -> limbs, compression, Montgomery groups), finish, t as
            # digits -> pinned host
            device.h2d_async(self.qu, self.h_qu, stream)
            self.ev_in.record(stream)
            self.side.wait_event(self.ev_in)
            device.h2d_async(self.d_ckd, self.h_ckd, self.side)
            self._seq("side_digits", self.side)
            self.ev_comp.record(self.side)
            self._gemv(stream, self.sms - self.ctas)
            stream.wait_event(self.ev_comp)
            self._seq("finish_digits", stream)
            device.d2h_async(self.h_td, self.d_td, stream)
        elif which == "e2e_g1":
            # respond(), graph 1 (main stream): query planes read straight from
            # the pinned (device-mapped) host qu -- no copy node -- then the GEMV
            if self.zero_copy:
                device.query_planes(self.h_qu.view(1, -1), 16, stream, planes=self.planes)
                device.umma_gemv(self.state.dbt, self.planes, 1, out=self.b, stream=stream,
                                 ctas=self.sms - self.ctas_e2e)
            else:
                device.h2d_async(self.qu, self.h_qu, stream)
                self._gemv(stream, self.sms - self.ctas_e2e)
        elif which in ("e2e_g2", "e2e_g2t", "w_g2t"):
            # respond() / respond_wire(), graph 2 (side stream): ck_o in (CPython
            # digits, or limb rows for the wire path), compression, Montgomery
            # groups; then (external wait for graph 1) the finish; e2e_g2 also
            # converts t to digits and copies it out, the others leave t in HBM
            if which == "w_g2t":
                device.h2d_async(self.cko, self.h_cko, stream)
            elif self.zero_copy:     # digits read from pinned host memory
                device.digits_to_limbs(self.h_ckd, self.kctx.lm, self.cko, stream)
            else:
                device.h2d_async(self.d_ckd, self.h_ckd, stream)
                device.digits_to_limbs(self.d_ckd, self.kctx.lm, self.cko, stream)
            self._compress(stream, self.ctas_e2e)
            self._groups_z(stream)
            device.stream_wait_event(stream, self.ev_gemv)
            if which == "e2e_g2":
                # t's digits written by the kernel straight into the pinned
                # (device-mapped) host buffer: no copy node at the tail
                self._finish(stream)
                if self.zero_copy:
                    device.limbs_to_digits(self.t, self.kctx.lm, self.h_td, stream)
                else:
                    device.limbs_to_digits(self.t, self.kctx.lm, self.d_td, stream)
                    device.d2h_async(self.h_td, self.d_td, stream)
            else:
                self._finish(stream)
        elif which == "side_limbs":
            # respond_wire(), side stream: ck_o limbs already staged
            self._compress(stream, self.ctas)
            self._groups_z(stream)
        elif which == "finish":
            self._finish(stream)
        elif which == "finish_digits":
            self._finish(stream)
            device.limbs_to_digits(self.t, self.kctx.lm, self.d_td, stream)
        elif which == "compress_digits":
            # respond(): ck_o arrives as CPython digits, t leaves as digits
            device.digits_to_limbs(self.d_ckd, self.kctx.lm, self.cko, stream)
            self._compress(stream, 0)
            self._groups_z(stream)
            self._finish(stream)
            device.limbs_to_digits(self.t, self.kctx.lm, self.d_td, stream)
        else:
            raise ValueError(which)

    # -- graph replay ----------------------------------------------------------

    def launch(self, which, stream):
        """Replay a captured graph with a raw cudaGraphLaunch (no torch stream
        context); the first call captures it through run()."""
        ex = self._exec.get(which) if USE_GRAPHS else None
        if ex is None:
            self.run(which, stream)
            if USE_GRAPHS:
                self._exec[which] = self.graphs[which].raw_cuda_graph_exec()
            return
        device.graph_launch(ex, stream)

    def run(self, which, stream):
        if self.key_m is None:
            self.set_key(self.kctx, stream)
        if not USE_GRAPHS:
            return self._seq(which, stream)
        g = self.graphs.get(which)
        if g is None:
            self._seq(which, stream)  # eager warm-up on the caller's stream
            stream.synchronize()
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(self.state.device)
            cap.wait_stream(stream)
            # thread_local: connection threads keep answering while one captures
            with _capture_lock, torch.cuda.graph(g, stream=cap,
                                                 capture_error_mode="thread_local"):
                self._seq(which, cap)
            stream.wait_stream(cap)
            self.graphs[which] = g
        with torch.cuda.stream(stream):
            g.replay()


def _mapped_in_place(t) -> bool:
    """The pinned host tensor's device alias is its own address."""
    import ctypes
    dev = ctypes.c_void_p()
    try:
        _lib.call("zpir_host_device_pointer", ctypes.c_void_p(t.data_ptr()), ctypes.byref(dev))
    except _lib.ZpirError:
        return False
    return dev.value == t.data_ptr()
