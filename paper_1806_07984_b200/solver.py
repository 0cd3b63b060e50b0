"""Time-step drivers on the GPU: the single-GPU replacement of the
reference's Algorithm-1 loop and of the enclave task
runtime.

DGSolver (uniform Cartesian or static adaptive mesh) and FVSolver keep all
state resident in HBM.  One step is a fixed sequence of kernel launches with
no host synchronisation -- dt is reduced and consumed on the device
(edg_dt_finalize) -- so a run of steps can be captured once into a CUDA
graph and replayed.

Uniform step (configs 1-3):   dt_finalize -> STP(all cells) -> fused
                              Riemann+corrector(+next-dt candidates)
Adaptive step (config 5), skeleton-first two-priority-stream schedule:
    main:    dt_finalize -> fork
    high:    STP(skeleton) -> faces/restrict of skeleton-only faces (incl. all hanging faces)
    low:     STP(enclave)
    main:    join -> faces of the remaining faces -> corrector(+dt)
FV step (config 4):           dt_finalize -> patch update(+next-dt candidates)
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .basis import get_basis
from .errors import ConfigError, EnclaveDgError, NumericalError
from .kernels import _check_supported, _stream, _torch
from .mesh import AdaptiveMesh, CartesianMesh
from .pde import PdeDescriptor


class KernelTimer:
    """CUDA-event pairs around named kernel launches on the launching stream."""

    def __init__(self):
        self.pairs = {}
        self._open = {}

    def begin(self, name):
        torch = _torch()
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream())
        self._open[name] = e

    def end(self, name):
        torch = _torch()
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream())
        self.pairs.setdefault(name, []).append((self._open.pop(name), e))

    def totals_ms(self):
        """{name: (launches, total ms)} -- call after a synchronize."""
        return {k: (len(v), sum(a.elapsed_time(b) for a, b in v)) for k, v in self.pairs.items()}


class _NativeGraph:
    """An executable CUDA graph instantiated by edg_graph_end."""

    def __init__(self, lib, exec_ptr, node_priorities):
        self.lib, self.exec = lib, exec_ptr
        self.node_priorities = node_priorities   # priority attribute of each kernel node

    def replay(self):
        _lib.check(self.lib.edg_graph_launch(self.exec, _stream()), "graph launch")

    def close(self):
        if self.exec is not None and self.exec.value:
            self.lib.edg_graph_destroy(self.exec)
        self.exec = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LaunchTrace:
    """Per-launch device timestamps of the step's kernels (edg_trace_next):
    slot i holds the global-timer ns of launch i's first CTA start and last
    CTA exit.  Labels (entity kind, stream, sweep) are recorded on the host
    when the launch is issued -- inside a graph capture they describe the
    captured nodes, and every replay rewrites the same slots.  The GPU
    analogue of the task trace of SPEC.md:392-400 (`record_trace`)."""

    def __init__(self, capacity: int = 512):
        torch = _torch()
        self.slots = torch.empty((capacity, 2), dtype=torch.int64, device="cuda")
        self.labels = []
        self.reset()

    def reset(self, labels: bool = False):
        """Re-arm every slot ({UINT64_MAX, 0}); optionally forget the labels."""
        self.slots[:, 0] = -1
        self.slots[:, 1] = 0
        if labels:
            self.labels = []

    def arm(self, lib, entity: str, worker: str, sweep: int):
        i = len(self.labels)
        if i >= self.slots.shape[0]:
            raise ConfigError("launch trace full")
        self.labels.append((entity, worker, sweep))
        _lib.check(lib.edg_trace_next(_lib.ptr(self.slots[i])), "trace")

    def records(self):
        """[(entity, worker, sweep, start_ns, end_ns)] -- call after a synchronize."""
        t = self.slots[:len(self.labels)].cpu().numpy().view(np.uint64)
        return [(e, w, sw, int(t[i, 0]), int(t[i, 1])) for i, (e, w, sw) in enumerate(self.labels)]


class _Base:
    def _common_alloc(self, max_steps):
        torch = self.torch
        self.dt = torch.zeros(1, dtype=torch.float64, device="cuda")
        self.dt_hist = torch.zeros(max_steps, dtype=torch.float64, device="cuda")
        self.slots = torch.empty(_lib.DT_SLOTS, dtype=torch.int64, device="cuda")
        self.status = torch.zeros(4, dtype=torch.int32, device="cuda")
        self.steps_done = 0
        self.max_steps = max_steps
        self._graph = None
        self._graph_steps = 0
        self._graph_key = None
        self.kernel_timer = None      # optional KernelTimer (events around the hot kernels)
        self.tracer = None            # optional LaunchTrace (per-launch device timestamps)

    def _trace(self, entity):
        """Arm the launch trace for the next launch (no-op without a tracer)."""
        if self.tracer is not None:
            self.tracer.arm(self.lib, entity, self._worker(), self.steps_done)

    def _worker(self):
        return "main"

    def _finalize_dt(self):
        """dt = cfl * min(candidates of the current state) (kernels.py:281);
        the device step counter status[2] indexes the dt history."""
        self._trace("DtFinalize")
        _lib.check(self.lib.edg_dt_finalize(_lib.ptr(self.slots), float(self.cfl), _lib.ptr(self.dt),
                                            _lib.ptr(self.dt_hist), -self.max_steps, _lib.ptr(self.status),
                                            _stream()), "dt_finalize")

    def check_status(self):
        st = self.status.cpu().numpy()
        if st[0] & 1:
            raise EnclaveDgError("no positive wave speed anywhere; cannot pick a time step")
        if st[0] & 2:
            raise AssertionError("face outcome missing (ordering bug)")
        if self.check_finite and st[1] > 0:
            raise NumericalError(f"{int(st[1])} cell(s) with a non-finite state")
        return st

    def dt_history(self):
        return self.dt_hist[:min(self.steps_done, self.max_steps)].cpu().numpy()

    # ------------------------------------------------------------- graphs --
    def run(self, steps: int, graph: bool = True, chunk: int = 2):
        """Advance `steps` steps.  With graph=True the launches of `chunk`
        consecutive steps are captured once into a CUDA graph and replayed
        (chunk must be even so the double buffers return to their roles)."""
        torch = self.torch
        self._state_gen = getattr(self, "_state_gen", 0) + 1
        if not graph:
            for _ in range(steps):
                self.step()
            return
        if chunk % 2:
            raise ConfigError("graph chunk must be even (ping-pong buffers)")
        full = steps // chunk
        if full and self.steps_done + full * chunk > self.max_steps:
            raise ConfigError("dt history too short: raise max_steps")
        if full:
            self.prepare_graph(chunk)
            for _ in range(full):
                self._graph.replay()
                self.steps_done += chunk
        for _ in range(steps - full * chunk):
            self.step()

    def prepare_graph(self, chunk: int = 2):
        """Capture `chunk` steps into a CUDA graph (once).  The graph bakes in
        which physical buffer holds the state, so it is re-captured when an
        odd number of eager steps has swapped the ping-pong roles.  Captured
        and instantiated through the C ABI (edg_graph_begin / edg_graph_end)
        so that the kernel nodes keep the priorities of the streams they were
        captured from (cudaGraphInstantiateFlagUseNodePriority): the
        skeleton-first schedule survives the graph."""
        torch = self.torch
        if chunk % 2:
            raise ConfigError("graph chunk must be even (ping-pong buffers)")
        key = (chunk, self.Q.data_ptr())
        if self._graph is not None and self._graph_key == key:
            return
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        steps0 = self.steps_done
        with torch.cuda.stream(side):
            _lib.check(self.lib.edg_graph_begin(_stream()), "graph capture")
            exc = None
            try:
                for _ in range(chunk):
                    self._enqueue_step()
                    self.steps_done += 1
            except BaseException as e:   # end the capture before re-raising
                exc = e
            ex = C.c_void_p()
            prios = (C.c_int32 * 1024)()
            nk = C.c_int32()
            st = self.lib.edg_graph_end(_stream(), C.byref(ex), prios, 1024, C.byref(nk))
            self.steps_done = steps0
            if exc is not None:
                if st == 0:
                    self.lib.edg_graph_destroy(ex)
                raise exc
            _lib.check(st, "graph instantiate")
        torch.cuda.current_stream().wait_stream(side)
        if self._graph is not None:
            self._graph.close()
        self._graph = _NativeGraph(self.lib, ex, list(prios[:min(nk.value, 1024)]))
        self._graph_steps, self._graph_key = chunk, key

    def step(self):
        self._state_gen = getattr(self, "_state_gen", 0) + 1
        self._enqueue_step()
        self.steps_done += 1

    # ------------------------------------------------- host-resident steps --
    def _auto_slabs(self, slabs):
        """Slab count of a streamed host step: the caller's, or about one slab
        per 4 MB of state, at most 64 -- a state of a few hundred KB goes as
        one slab (every slab costs its own copies and launches: config 1's
        93 KB took 2.1 ms per step in 16 slabs, 0.17 ms in one), a large one
        in many (the upload of step k + 1 trails the download of step k by one
        slab: config 3, 1.31 GB, 29.5 / 28.9 / 28.3 ms per step in 16 / 32 /
        64 slabs)."""
        if slabs is not None:
            return int(slabs)
        nbytes = self.Q.numel() * self.Q.element_size()
        return int(max(1, min(64, nbytes // (4 << 20))))

    def _host_stream(self, q_in, q_out, bounds, order, npts, plan):
        """One step from the host buffer q_in to the host buffer q_out,
        streamed in slabs (cell / patch ranges `bounds`):

            copy-in stream : H2D slab j          (waits for D2H slab j of the previous call)
            current stream : dt candidates of slab j as it lands -> dt = cfl * min
                             -> plan[i]() enqueues kernels, returns the slabs now final
            copy-out stream: D2H of each final slab

        dt is the admissible step of q_in itself (kernels.py:267-281), so the
        result is bitwise that of set_state(q_in); step().  q_in / q_out: CPU
        tensors of the state's shape (pinned for asynchronous copies).  q_out
        is complete when the event `host_ready` has completed (host_wait()
        makes the current stream wait for it); the current stream does not
        wait, so the next call's uploads overlap this call's downloads, and
        back-to-back calls only wait per slab for the previous call's download
        of the same slab (other work on the state in between makes the uploads
        wait for the current stream)."""
        torch = self.torch
        lib = self.lib
        if not hasattr(self, "_sh"):
            self._sh = {"in": torch.cuda.Stream(), "out": torch.cuda.Stream(), "prev_out": {}}
        sh = self._sh
        src = q_in.reshape(self.Q.shape)
        dst = q_out.reshape(self.Q.shape)
        main = torch.cuda.current_stream()
        Q, Qn = self.Q, self.Qn
        if sh.get("gen") != getattr(self, "_state_gen", 0):
            sh["in"].wait_stream(main)
            sh["prev_out"] = {}
        _lib.check(lib.edg_dt_slots_reset(_lib.ptr(self.slots), _stream()), "dt reset")
        for j in range(len(bounds) - 1):
            c0, c1 = bounds[j], bounds[j + 1]
            with torch.cuda.stream(sh["in"]):
                prev = sh["prev_out"].get((c0, c1))
                if prev is not None:
                    sh["in"].wait_event(prev)     # host / device slab still being read by the last call's copy-out
                Q[c0:c1].copy_(src[c0:c1], non_blocking=True)
                e = torch.cuda.Event()
                e.record(sh["in"])
            main.wait_event(e)
            _lib.check(lib.edg_cell_speed_reduce(C.byref(self.native), order, c1 - c0, npts, _lib.ptr(Q[c0:c1]),
                                                 _lib.ptr(self.hmin), 0, _lib.ptr(self.slots), _stream()),
                       "admissible_dt")
        self._finalize_dt()
        prev_out = {}
        for run in plan:
            for c in run():
                c0, c1 = bounds[c], bounds[c + 1]
                e = torch.cuda.Event()
                e.record(main)
                with torch.cuda.stream(sh["out"]):
                    sh["out"].wait_event(e)
                    dst[c0:c1].copy_(Qn[c0:c1], non_blocking=True)
                    eo = torch.cuda.Event()
                    eo.record(sh["out"])
                prev_out[(c0, c1)] = eo
        sh["prev_out"] = prev_out
        sh["gen"] = getattr(self, "_state_gen", 0)
        self.host_ready = torch.cuda.Event()
        self.host_ready.record(sh["out"])
        self.Q, self.Qn = self.Qn, self.Q
        self.steps_done += 1

    def host_wait(self):
        """Make the current stream wait for the last step_host's downloads."""
        ev = getattr(self, "host_ready", None)
        if ev is not None:
            self.torch.cuda.current_stream().wait_event(ev)


class DGSolver(_Base):
    """ADER-DG time stepping on the GPU (Algorithm 1 semantics)."""

    # the predictor's work order (cells sorted by their last Picard count so
    # that CTAs are homogeneous) only matters once the cells outnumber the
    # resident predictor slots; below this the three ordering launches cost
    # more than they save (config 1: 729 cells, 19 us per step, 6 launches)
    ORDER_MIN_CELLS = 8192

    def __init__(self, pde: PdeDescriptor, order: int, mesh, cfl: float, tol: float = 1e-10, max_iter=None,
                 check_finite: bool = True, max_steps: int = 4096, two_streams: bool = True):
        torch = self.torch = _torch()
        self.lib = _lib.load()
        _check_supported(pde, order)
        self.pde, self.order, self.mesh, self.cfl = pde, order, mesh, float(cfl)
        self.tol = float(tol)
        self.max_iter = 0 if max_iter is None else int(max_iter)
        self.check_finite = check_finite
        self.basis = get_basis(order)
        self.table = self.basis.device_table()
        self.native = pde.native()
        if mesh.dim != pde.dim:
            raise ConfigError("mesh and pde dimension differ")
        self.iter_total = torch.zeros(1, dtype=torch.int64, device="cuda")   # sum of Picard iterations
        self._common_alloc(max_steps)
        self.adaptive = isinstance(mesh, AdaptiveMesh)
        self._cap = (0, 0)        # allocated (cells, outcome rows)
        self.two_streams = two_streams
        if self.adaptive and two_streams:
            lo, hi = C.c_int32(), C.c_int32()
            _lib.check(self.lib.edg_stream_priority_range(C.byref(lo), C.byref(hi)), "priority range")
            try:
                self.s_hi = torch.cuda.Stream(priority=hi.value)
            except (RuntimeError, ValueError):
                self.s_hi = torch.cuda.Stream(priority=-1)
            self.s_lo = torch.cuda.Stream(priority=lo.value)
        self._load_mesh(mesh)

    def _load_mesh(self, mesh):
        """Mesh-dependent device tables and per-cell / per-face buffers.  The
        buffers are views of allocations that only grow (by 1/4 headroom), so a
        remesh within the capacity reallocates nothing."""
        torch = self.torch
        d, m, n = self.pde.dim, self.pde.m, self.basis.n
        self.mesh = mesh
        Cn = self.ncells = mesh.ncells
        nout = (mesh.nleaf + mesh.nparent) if self.adaptive else 0
        f64 = dict(dtype=torch.float64, device="cuda")
        cap_c, cap_o = self._cap
        if Cn > cap_c:
            cap_c = Cn if cap_c == 0 else max(Cn, cap_c + cap_c // 4)
            self._buf = {k: torch.zeros((cap_c,) + shp, **f64) for k, shp in
                         (("Q", (m,) + (n,) * d), ("Qn", (m,) + (n,) * d), ("q_end", (m,) + (n,) * d),
                          ("trace_q", (2 * d, m) + (n,) * (d - 1)), ("trace_f", (2 * d, m) + (n,) * (d - 1)))}
            self._buf["iterations"] = torch.zeros(cap_c, dtype=torch.int32, device="cuda")
            self._buf["converged"] = torch.zeros(cap_c, dtype=torch.uint8, device="cuda")
        if nout > cap_o:
            cap_o = nout if cap_o == 0 else max(nout, cap_o + cap_o // 4)
            self._buf["outcomes"] = torch.zeros((cap_o, m) + (n,) * (d - 1), **f64)
        self._cap = (cap_c, cap_o)
        for k in ("Q", "Qn", "q_end", "trace_q", "trace_f", "iterations", "converged"):
            setattr(self, k, self._buf[k][:Cn])
        i32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()  # noqa: E731
        i8 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int8)).cuda()  # noqa: E731
        self._graph = None            # the graph bakes in the buffers and tables
        if self.adaptive:
            self.edges = torch.from_numpy(mesh.edges.copy()).cuda()
            self.edges_per_cell = 1
            self.hmin = torch.from_numpy(mesh.hmin.copy()).cuda()
            self.face_axis = i32(mesh.face_axis)
            self.face_cell = i32(mesh.face_cell)
            self.face_kind = i8(mesh.face_kind)
            self.face_cp = i8(mesh.face_child_pos)
            self.face_vpath = i8(mesh.face_vpath)
            self.face_vdepth = i8(mesh.face_vdepth)
            self.max_chain = int(mesh.max_chain)
            self.outcome_cp = i8(mesh.outcome_cp)
            self.side_face = i32(mesh.side_face)
            self.outcomes = self._buf["outcomes"][:nout]
            self.skel = i32(mesh.skeleton)
            self.encl = i32(mesh.enclave)
            self.parent_face = i32(mesh.parent_face)
            self.parent_children = i32(mesh.parent_children)
            self.parent_groups = [tuple(g) for g in mesh.parent_groups]
            self.nface_sk = mesh.nleaf_skeleton
        else:
            self.edges = torch.tensor([mesh.h] * d, **f64)
            self.edges_per_cell = 0
            self.hmin = torch.tensor([mesh.h], **f64)
            self.nbr = i32(mesh.nbr)
            # predictor work order: cells sorted by their last Picard count
            self.work_order = torch.arange(Cn, dtype=torch.int32, device="cuda")
            self.order_scratch = torch.zeros(128, dtype=torch.int32, device="cuda")

    def remesh(self, mesh, Q):
        """Adopt an adapted mesh of the same kind in place (dynamic AMR without
        a new solver): device tables rebuilt, buffers reused while they fit,
        the state `Q` (new cell order) installed, the CUDA graph dropped."""
        if isinstance(mesh, AdaptiveMesh) != self.adaptive or mesh.dim != self.pde.dim:
            raise ConfigError("remesh needs a mesh of the same kind and dimension")
        self.torch.cuda.current_stream().synchronize()   # in-flight work still reads the old tables
        self._load_mesh(mesh)
        self.set_state(Q)

    # ---------------------------------------------------------------- state --
    def set_state(self, Q):
        torch = self.torch
        src = Q if isinstance(Q, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(Q, dtype=np.float64))
        self.Q.copy_(src.reshape(self.Q.shape), non_blocking=True)
        self.steps_done = 0
        self._state_gen = getattr(self, "_state_gen", 0) + 1
        self.status.zero_()
        self._seed_dt()

    def _seed_dt(self):
        """Candidates of the current state (the corrector refreshes them every step)."""
        lib = self.lib
        _lib.check(lib.edg_dt_slots_reset(_lib.ptr(self.slots), _stream()), "dt reset")
        npts = self.basis.n ** self.pde.dim
        _lib.check(lib.edg_cell_speed_reduce(C.byref(self.native), self.order, self.ncells, npts, _lib.ptr(self.Q),
                                             _lib.ptr(self.hmin), self.edges_per_cell, _lib.ptr(self.slots),
                                             _stream()), "admissible_dt")

    def state(self):
        return self.Q

    # ------------------------------------------------------- slab helpers --
    def _slab_bounds(self, slabs):
        """Cell ranges of `slabs` runs of whole axis-0 layers (uniform grid)."""
        N, d = self.mesh.N, self.pde.dim
        S = max(1, min(int(slabs), N))
        layer = N ** (d - 1)
        return [(N * j // S) * layer for j in range(S + 1)]

    def _slab_order_stp(self, Q, order, c0, c1, background=False, entity="STP"):
        """Picard order of cells [c0, c1) by their last iteration counts,
        then the predictor over them (slab-local indices, offset buffers)."""
        lib, nc = self.lib, c1 - c0
        _lib.check(lib.edg_order_by_iterations(nc, _lib.ptr(self.iterations[c0:c1]), _lib.ptr(order[c0:c1]),
                                               _lib.ptr(self.order_scratch), _stream()), "order")
        self._trace(entity)
        fn = lib.edg_stp_picard_background if background else lib.edg_stp_picard
        _lib.check(fn(C.byref(self.native), self.order, _lib.ptr(self.table), _lib.ptr(Q[c0:c1]),
                      _lib.ptr(order[c0:c1]), nc, _lib.ptr(self.edges), 0, _lib.ptr(self.dt), self.tol,
                      self.max_iter, _lib.ptr(self.q_end[c0:c1]), None, _lib.ptr(self.trace_q[c0:c1]),
                      _lib.ptr(self.trace_f[c0:c1]), _lib.ptr(self.iterations[c0:c1]),
                      _lib.ptr(self.converged[c0:c1]), _lib.ptr(self.iter_total), _stream()), "stp_picard")

    def _slab_corrector(self, Qn, c0, c1):
        self._trace("Corrector")
        _lib.check(self.lib.edg_corrector_grid_range(
            C.byref(self.native), self.order, _lib.ptr(self.table), self.mesh.N, int(self.mesh.periodic), c0, c1 - c0,
            _lib.ptr(self.q_end), _lib.ptr(self.trace_q), _lib.ptr(self.trace_f), _lib.ptr(self.edges), _lib.ptr(Qn),
            _lib.ptr(self.slots), _lib.ptr(self.hmin), _lib.ptr(self.status), _stream()), "corrector")

    def _corrector_schedule(self, S):
        """[(slab whose predictor completes, [slabs correctable right after])]:
        slab j reads the traces of slabs j - 1 and j + 1 (wrapping on a
        periodic grid, where slab 0 is corrected last)."""
        per = self.mesh.periodic and S > 1
        pending = list(range(1, S)) + [0] if per else list(range(S))
        done, out = set(), []
        for j in range(S):
            done.add(j)
            ready = []
            while pending:
                c = pending[0]
                need = {(c - 1) % S, c, (c + 1) % S} if per else {x for x in (c - 1, c, c + 1) if 0 <= x < S}
                if not need <= done:
                    break
                ready.append(pending.pop(0))
            out.append((j, ready))
        return out

    def _slab_order_buf(self):
        if getattr(self, "_slab_order", None) is None or self._slab_order.numel() < self.ncells:
            self._slab_order = self.torch.zeros(self.ncells, dtype=self.torch.int32, device="cuda")
        return self._slab_order

    # ------------------------------------------------- host-resident steps --
    def step_host(self, q_in, q_out, slabs=None):
        """One step from a host state to a host buffer (the drop-in use of
        the reference's numpy API, where every call takes and returns host
        arrays), streamed in slabs of the uniform grid (_Base._host_stream):
        once every slab has landed and dt is reduced, the predictor of slab j
        is followed by the corrector of slab j - 1 (its face neighbours lie in
        slabs j - 2 .. j; on a periodic grid slab 0 is corrected last) and that
        slab's download.  Bitwise set_state(q_in); step()."""
        if self.adaptive:
            raise ConfigError("step_host streams uniform grids only")
        bounds = self._slab_bounds(self._auto_slabs(slabs))
        order = self._slab_order_buf()
        Q, Qn = self.Q, self.Qn
        plan = []
        for j, ready in self._corrector_schedule(len(bounds) - 1):
            def run(j=j, ready=ready):
                self._slab_order_stp(Q, order, bounds[j], bounds[j + 1])
                for c in ready:
                    self._slab_corrector(Qn, bounds[c], bounds[c + 1])
                return ready
            plan.append(run)
        self._host_stream(q_in, q_out, bounds, self.order, self.basis.n ** self.pde.dim, plan)

    # ----------------------------------------------------------------- step --
    def _worker(self):
        if self.adaptive and self.two_streams:
            cur = self.torch.cuda.current_stream()
            if cur == self.s_hi:
                return "hi"
            if cur == self.s_lo:
                return "lo"
        return "main"

    def _stp(self, cell_list, nwork, entity="STP", background=False):
        self._trace(entity)
        fn = self.lib.edg_stp_picard_background if background else self.lib.edg_stp_picard
        return fn(C.byref(self.native), self.order, _lib.ptr(self.table), _lib.ptr(self.Q),
                                       _lib.ptr(cell_list), nwork, _lib.ptr(self.edges), self.edges_per_cell,
                                       _lib.ptr(self.dt), self.tol, self.max_iter, _lib.ptr(self.q_end), None,
                                       _lib.ptr(self.trace_q), _lib.ptr(self.trace_f), _lib.ptr(self.iterations),
                                       _lib.ptr(self.converged), _lib.ptr(self.iter_total), _stream())

    def _faces(self, off, cnt, entity="Faces"):
        """Rusanov on leaf faces [off, off + cnt) (skeleton-only faces come first);
        a virtual side is the coarse owner's trace interpolated along the
        leaf's chain path."""
        if cnt <= 0:
            return
        sl = slice(off, off + cnt)
        self._trace(entity)
        _lib.check(self.lib.edg_faces_rusanov_chain(C.byref(self.native), self.order, _lib.ptr(self.table), cnt,
                                                    _lib.ptr(self.face_axis[sl]), _lib.ptr(self.face_cell[sl]),
                                                    _lib.ptr(self.face_kind[sl]), _lib.ptr(self.face_vpath[sl]),
                                                    _lib.ptr(self.face_vdepth[sl]), int(self.face_vpath.shape[1]),
                                                    _lib.ptr(self.trace_q), _lib.ptr(self.outcomes[sl]),
                                                    _stream()), "faces_rusanov")

    def _restrict(self):
        """Parent outcomes restricted from their children, one launch per
        level of the face forest, deepest first (a parent of a parent reads
        complete children)."""
        for g0, gn in self.parent_groups:
            self._trace("Restrict")
            _lib.check(self.lib.edg_faces_restrict(self.pde.dim, self.pde.m, self.order, _lib.ptr(self.table), gn,
                                                   _lib.ptr(self.parent_face[g0:g0 + gn]),
                                                   _lib.ptr(self.parent_children[g0:g0 + gn]),
                                                   _lib.ptr(self.outcome_cp), _lib.ptr(self.outcomes), _stream()),
                       "faces_restrict")

    def _enqueue_step(self):
        torch = self.torch
        lib = self.lib
        self._finalize_dt()
        tm = self.kernel_timer
        if not self.adaptive:
            if tm:
                tm.begin("stp")
            _lib.check(self._stp(self.work_order, self.ncells), "stp_picard")
            if tm:
                tm.end("stp")
                tm.begin("corrector")
            self._trace("Corrector")
            _lib.check(lib.edg_corrector_grid(C.byref(self.native), self.order, _lib.ptr(self.table), self.mesh.N,
                                              int(self.mesh.periodic), _lib.ptr(self.q_end), _lib.ptr(self.trace_q),
                                              _lib.ptr(self.trace_f), _lib.ptr(self.edges), _lib.ptr(self.Qn),
                                              _lib.ptr(self.slots), _lib.ptr(self.hmin), _lib.ptr(self.status),
                                              _stream()), "corrector")
            if tm:
                tm.end("corrector")
            if self.ncells >= self.ORDER_MIN_CELLS:
                _lib.check(lib.edg_order_by_iterations(self.ncells, _lib.ptr(self.iterations),
                                                       _lib.ptr(self.work_order), _lib.ptr(self.order_scratch),
                                                       _stream()), "order")
        else:
            nsk, F = self.nface_sk, self.mesh.nleaf

            def skeleton_phase():
                _lib.check(self._stp(self.skel, int(self.skel.numel()), "SkeletonSTP"), "stp_picard(skeleton)")
                self._faces(0, nsk, "SkeletonFaces")
                self._restrict()

            def enclave_phase(background=False):
                _lib.check(self._stp(self.encl, int(self.encl.numel()), "EnclaveSTP", background),
                           "stp_picard(enclave)")

            if tm is not None:
                # timed (benchmark) order on one stream -- all predictors, then
                # the faces: same results bitwise, the events bracket the kernels
                tm.begin("stp")
                _lib.check(self._stp(self.skel, int(self.skel.numel()), "SkeletonSTP"), "stp_picard(skeleton)")
                _lib.check(self._stp(self.encl, int(self.encl.numel()), "EnclaveSTP"), "stp_picard(enclave)")
                tm.end("stp")
                self._faces(0, nsk, "SkeletonFaces")
                self._restrict()
            elif self.two_streams:
                main = torch.cuda.current_stream()
                self.s_hi.wait_stream(main)
                self.s_lo.wait_stream(main)
                with torch.cuda.stream(self.s_hi):
                    skeleton_phase()
                with torch.cuda.stream(self.s_lo):
                    enclave_phase(background=True)
                main.wait_stream(self.s_hi)
                main.wait_stream(self.s_lo)
            else:
                skeleton_phase()
                enclave_phase()
            self._faces(nsk, F - nsk)
            if tm:
                tm.begin("corrector")
            self._trace("Corrector")
            _lib.check(lib.edg_corrector(C.byref(self.native), self.order, _lib.ptr(self.table), self.ncells,
                                         _lib.ptr(self.q_end), _lib.ptr(self.trace_q), _lib.ptr(self.trace_f),
                                         None, _lib.ptr(self.side_face), _lib.ptr(self.outcomes),
                                         _lib.ptr(self.edges), self.edges_per_cell, _lib.ptr(self.Qn),
                                         _lib.ptr(self.slots), _lib.ptr(self.hmin), _lib.ptr(self.status),
                                         _stream()), "corrector")
            if tm:
                tm.end("corrector")
        self.Q, self.Qn = self.Qn, self.Q


class FVSolver(_Base):
    """Patch finite-volume stepping (config 4): patches (B, m, k^3) of a
    Cartesian patch grid, outflow boundaries."""

    def __init__(self, pde: PdeDescriptor, cells_per_axis: int, k: int, cfl: float, periodic: bool = False,
                 check_finite: bool = True, max_steps: int = 4096):
        torch = self.torch = _torch()
        self.lib = _lib.load()
        if cells_per_axis % k:
            raise ConfigError("cells per axis must be a multiple of the patch size")
        self.pde, self.k, self.cfl = pde, k, float(cfl)
        self.check_finite = check_finite
        self.native = pde.native()
        d, m = pde.dim, pde.m
        npx = cells_per_axis // k
        self.pmesh = CartesianMesh(npx, d, periodic)
        self.npatches = self.pmesh.ncells
        self.h_cell = 1.0 / cells_per_axis
        f64 = dict(dtype=torch.float64, device="cuda")
        self.Q = torch.zeros((self.npatches, m) + (k,) * d, **f64)
        self.Qn = torch.zeros_like(self.Q)
        self.nbr = torch.from_numpy(self.pmesh.nbr.copy()).cuda()
        self.edges = torch.tensor([self.h_cell * k] * d, **f64)
        self.hmin = torch.tensor([self.h_cell], **f64)
        self._common_alloc(max_steps)

    def set_state(self, P):
        torch = self.torch
        src = P if isinstance(P, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(P, dtype=np.float64))
        self.Q.copy_(src.reshape(self.Q.shape), non_blocking=True)
        self.steps_done = 0
        self._state_gen = getattr(self, "_state_gen", 0) + 1
        self.status.zero_()
        _lib.check(self.lib.edg_dt_slots_reset(_lib.ptr(self.slots), _stream()), "dt reset")
        _lib.check(self.lib.edg_cell_speed_reduce(C.byref(self.native), 0, self.npatches, self.k ** self.pde.dim,
                                                  _lib.ptr(self.Q), _lib.ptr(self.hmin), 0, _lib.ptr(self.slots),
                                                  _stream()), "admissible_dt")

    def state(self):
        return self.Q

    def step_host(self, q_in, q_out, slabs=None):
        """One step from a host state to a host buffer, streamed in slabs of
        patch layers (_Base._host_stream): once every slab has landed and dt
        is reduced, each slab's patch update (its halos are read from the
        uploaded neighbour patches) is followed by that slab's download.
        Bitwise set_state(q_in); step()."""
        N, d = self.pmesh.N, self.pde.dim
        S = max(1, min(int(self._auto_slabs(slabs)), N))
        layer = N ** (d - 1)
        bounds = [(N * j // S) * layer for j in range(S + 1)]
        Q, Qn, lib = self.Q, self.Qn, self.lib
        plan = []
        for j in range(S):
            def run(j=j):
                self._trace("FVPatch")
                _lib.check(lib.edg_fv_grid_step_range(C.byref(self.native), self.k, N, int(self.pmesh.periodic),
                                                      bounds[j], bounds[j + 1] - bounds[j], _lib.ptr(Q),
                                                      _lib.ptr(self.dt), _lib.ptr(self.edges), _lib.ptr(Qn),
                                                      _lib.ptr(self.slots), self.h_cell, _lib.ptr(self.status),
                                                      _stream()), "fv_patch_step")
                return [j]
            plan.append(run)
        self._host_stream(q_in, q_out, bounds, 0, self.k ** d, plan)

    def _enqueue_step(self):
        lib = self.lib
        self._finalize_dt()
        tm = self.kernel_timer
        if tm:
            tm.begin("fv")
        self._trace("FVPatch")
        _lib.check(lib.edg_fv_grid_step(C.byref(self.native), self.k, self.pmesh.N, int(self.pmesh.periodic),
                                        _lib.ptr(self.Q), _lib.ptr(self.dt), _lib.ptr(self.edges),
                                        _lib.ptr(self.Qn), _lib.ptr(self.slots), self.h_cell,
                                        _lib.ptr(self.status), _stream()), "fv_patch_step")
        if tm:
            tm.end("fv")
        self.Q, self.Qn = self.Qn, self.Q
