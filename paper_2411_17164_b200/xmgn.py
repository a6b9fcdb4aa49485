"""Thin ctypes binding of libxmgn.so (include/xmgn.h) -- argument marshalling only.

Every step of the processor runs in the CUDA library; this module converts
numpy / torch arguments to pointers and status codes to exceptions.  There is
no fallback: if libxmgn.so is missing the import fails.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("XMGN_LIB_OVERRIDE", os.path.join(_HERE, "libxmgn.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
_lib = ctypes.CDLL(LIB_PATH)

PREC_BF16, PREC_FP32_CHECK, PREC_FP16 = 0, 1, 2
STATUS = {0: "OK", 1: "EINVAL", 2: "EHALO", 3: "ESTATE", 4: "ENOMEM", 5: "ECUDA", 6: "ENCCL",
          7: "ENONFINITE", 8: "EUNSUPPORTED"}


class XmgnError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = STATUS.get(status, status)


_vp, _i64, _i32, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t


class GraphDesc(ctypes.Structure):
    _fields_ = [("n_nodes", _i64), ("n_edges", _i64), ("csr_offsets", _vp), ("csr_sources", _vp),
                ("n_parts", ctypes.c_int32), ("halo_depth", ctypes.c_int32), ("owned_offsets", _vp),
                ("owned", _vp), ("halo_offsets", _vp), ("halo", _vp), ("halo_ring", _vp)]


class PartInfo(ctypes.Structure):
    _fields_ = [("n_owned", _i64), ("n_local", _i64), ("e_local", _i64), ("depth", ctypes.c_int32),
                ("ring_nodes", _i64 * 65), ("ring_edges", _i64 * 65)]


class ModelCfg(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_int32), ("layers", ctypes.c_int32), ("mlp_hidden_layers", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("ln_eps", ctypes.c_float)]


class AdamCfg(ctypes.Structure):
    _fields_ = [("lr_max", ctypes.c_float), ("lr_min", ctypes.c_float), ("total_steps", _i64),
                ("beta1", ctypes.c_float), ("beta2", ctypes.c_float), ("eps", ctypes.c_float),
                ("clip", ctypes.c_float)]


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype, f.argtypes = res, args
    return f


_sig("xmgn_last_error", ctypes.c_char_p, [])
_sig("xmgn_version", ctypes.c_char_p, [])
_sig("xmgn_load_graph", _i32, [ctypes.POINTER(GraphDesc), _i32, ctypes.POINTER(_vp)])
_sig("xmgn_part_info_get", _i32, [_vp, _i32, ctypes.POINTER(PartInfo)])
_sig("xmgn_export_part", _i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp])
_sig("xmgn_free_graph", None, [_vp])
_sig("xmgn_param_count", _sz, [ctypes.POINTER(ModelCfg)])
_sig("xmgn_workspace_create", _i32, [_vp, ctypes.POINTER(ModelCfg), ctypes.POINTER(_vp)])
_sig("xmgn_workspace_create_infer", _i32, [_vp, ctypes.POINTER(ModelCfg), ctypes.POINTER(_vp)])
_sig("xmgn_workspace_bytes", _sz, [_vp])
_sig("xmgn_workspace_free", None, [_vp])
_sig("xmgn_processor_fwd", _i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp])
_sig("xmgn_processor_bwd", _i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp])
_sig("xmgn_check_finite", _i32, [_vp, _sz, _vp])
_sig("xmgn_comm_unique_id", _i32, [ctypes.c_char_p])
_sig("xmgn_comm_init", _i32, [ctypes.c_char_p, _i32, _i32, _i32, ctypes.POINTER(_vp)])
_sig("xmgn_grad_reduce", _i32, [_vp, _vp, _sz, _vp])
_sig("xmgn_comm_destroy", None, [_vp])
_sig("xmgn_gather_rows", _i32, [_vp, _vp, _i64, _i64, _vp, _vp, _vp])
_sig("xmgn_scatter_rows", _i32, [_vp, _vp, _i64, _i64, _vp, _vp])
_sig("xmgn_cosine_lr", ctypes.c_float, [ctypes.POINTER(AdamCfg), _i64])
_sig("xmgn_adam_step", _i32, [ctypes.POINTER(AdamCfg), _i64, _vp, _vp, _vp, _vp, _sz, ctypes.c_float, _vp, _vp])
_sig("xmgn_selftest_gemm", _i32, [_i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp])
_sig("xmgn_io_param_count", _sz, [ctypes.POINTER(ModelCfg)])
_sig("xmgn_model_fwd", _i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp])
_sig("xmgn_model_bwd", _i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp])
_sig("xmgn_build_graph", _i32, [_vp, _i64, _vp, _i32, _i32, _i32, _i32, _i32, _vp, ctypes.POINTER(_vp)])
_sig("xmgn_built_graph_desc", _i32, [_vp, ctypes.POINTER(GraphDesc)])
_sig("xmgn_built_graph_owner", _i32, [_vp, _vp])
_sig("xmgn_built_graph_free", None, [_vp])
_sig("xmgn_launch_count", ctypes.c_longlong, [])
_sig("xmgn_profile_enable", _i32, [_i32])
_sig("xmgn_profile_collect", _i32, [ctypes.c_char_p, _sz, ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_longlong), _i32, ctypes.POINTER(_i32)])

EXPORTS = ["xmgn_last_error", "xmgn_version", "xmgn_load_graph", "xmgn_part_info_get", "xmgn_export_part",
           "xmgn_free_graph", "xmgn_param_count", "xmgn_workspace_create", "xmgn_workspace_create_infer",
           "xmgn_workspace_bytes",
           "xmgn_workspace_free", "xmgn_processor_fwd", "xmgn_processor_bwd", "xmgn_check_finite",
           "xmgn_comm_unique_id", "xmgn_comm_init", "xmgn_grad_reduce", "xmgn_comm_destroy", "xmgn_gather_rows",
           "xmgn_scatter_rows",
           "xmgn_io_param_count", "xmgn_model_fwd", "xmgn_model_bwd",
           "xmgn_build_graph", "xmgn_built_graph_desc", "xmgn_built_graph_owner", "xmgn_built_graph_free",
           "xmgn_cosine_lr", "xmgn_adam_step", "xmgn_selftest_gemm", "xmgn_launch_count", "xmgn_profile_enable", "xmgn_profile_collect"]


def _check(status):
    if status != 0:
        raise XmgnError(status, _lib.xmgn_last_error().decode(errors="replace"))


def version():
    return _lib.xmgn_version().decode()


def _ptr(x):
    """Device/host pointer of a torch tensor or numpy array (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _stream(s):
    if s is None:
        return None
    return getattr(s, "cuda_stream", s)


def _i64c(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class Graph:
    """xmgn_load_graph: CSR by destination + per-partition owned / halo lists."""

    def __init__(self, offsets, sources, owned_offsets, owned, halo_offsets, halo, halo_ring, halo_depth,
                 device=0):
        self._keep = [_i64c(offsets), _i64c(sources), _i64c(owned_offsets), _i64c(owned), _i64c(halo_offsets),
                      _i64c(halo), np.ascontiguousarray(halo_ring, dtype=np.int32)]
        o, s, oo, ow, ho, ha, hr = self._keep
        d = GraphDesc(len(o) - 1, len(s), o.ctypes.data, s.ctypes.data, len(oo) - 1, int(halo_depth),
                      oo.ctypes.data, ow.ctypes.data, ho.ctypes.data, ha.ctypes.data, hr.ctypes.data)
        h = _vp()
        _check(_lib.xmgn_load_graph(ctypes.byref(d), int(device), ctypes.byref(h)))
        self.handle = h
        self.n_parts = len(oo) - 1
        self.device = int(device)
        self._keep = None

    @classmethod
    def from_bundle(cls, b, halo_depth, device=0):
        return cls(b["offsets"], b["sources"], b["owned_offsets"], b["owned"], b["halo_offsets"], b["halo"],
                   b["halo_ring"], halo_depth, device)

    def part_info(self, p):
        pi = PartInfo()
        _check(_lib.xmgn_part_info_get(self.handle, int(p), ctypes.byref(pi)))
        d = pi.depth
        return dict(n_owned=pi.n_owned, n_local=pi.n_local, e_local=pi.e_local, depth=d,
                    ring_nodes=list(pi.ring_nodes[:d + 2]), ring_edges=list(pi.ring_edges[:d + 2]))

    def export(self, p):
        info = self.part_info(p)
        n, e = info["n_local"], info["e_local"]
        out = dict(gid=np.empty(n, np.int64), offsets=np.empty(n + 1, np.int64), sources=np.empty(e, np.int64),
                   edge_gid=np.empty(e, np.int64), rev=np.empty(e, np.int64))
        _check(_lib.xmgn_export_part(self.handle, int(p), out["gid"].ctypes.data, out["offsets"].ctypes.data,
                                     out["sources"].ctypes.data, out["edge_gid"].ctypes.data,
                                     out["rev"].ctypes.data))
        out.update(info)
        return out

    def close(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.xmgn_free_graph(self.handle)
        self.handle = None

    def __del__(self):
        self.close()


def build_graph(pos, level_counts, k, n_parts, halo_depth, stream=None):
    """xmgn_build_graph (NEXT-4): the multi-scale kNN graph, RCB partitions and halo lists of a
    device FP32 [n, 3] point cloud, returned as a bundle dict of numpy arrays (the layout of
    xmgn_inputs.configs.build) -- every step runs on the GPU."""
    n = int(pos.shape[0])
    dv = pos.device.index
    lc = _i64c(level_counts)
    h = _vp()
    _check(_lib.xmgn_build_graph(_dev_f32(pos, "pos", 3 * n), n, lc.ctypes.data, len(lc), int(k), int(n_parts),
                                 int(halo_depth), dv, _stream(stream), ctypes.byref(h)))
    try:
        d = GraphDesc()
        _check(_lib.xmgn_built_graph_desc(h, ctypes.byref(d)))
        P = d.n_parts

        def arr(ptr, count, dt):
            if count == 0:
                return np.zeros(0, dt)
            ct = ctypes.c_int64 if dt == np.int64 else ctypes.c_int32
            return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ct)), shape=(count,)).astype(dt).copy()

        oo = arr(d.owned_offsets, P + 1, np.int64)
        ho = arr(d.halo_offsets, P + 1, np.int64)
        out = dict(offsets=arr(d.csr_offsets, n + 1, np.int64), sources=arr(d.csr_sources, d.n_edges, np.int64),
                   owned_offsets=oo, owned=arr(d.owned, int(oo[-1]), np.int64), halo_offsets=ho,
                   halo=arr(d.halo, int(ho[-1]), np.int64), halo_ring=arr(d.halo_ring, int(ho[-1]), np.int32))
        owner = np.empty(n, np.int64)
        _check(_lib.xmgn_built_graph_owner(h, owner.ctypes.data))
        out["owner"] = owner
        return out
    finally:
        _lib.xmgn_built_graph_free(h)


def model_cfg(hidden, layers, m=2, precision=PREC_FP16, ln_eps=1e-5):
    return ModelCfg(hidden, layers, m, precision, ln_eps)


def param_count(cfg):
    return int(_lib.xmgn_param_count(ctypes.byref(cfg)))


def io_param_count(cfg):
    return int(_lib.xmgn_io_param_count(ctypes.byref(cfg)))


IO_NSTATS, IO_DOUT = 56, 4   # [mean | std] of the 24 node + 4 edge inputs; outputs per node


def _dev_f32(t, name, numel, device=None):
    """Device pointer of a CUDA, float32, contiguous torch tensor holding at least
    `numel` values (the library reads / writes exactly that many)."""
    if t is None:
        return None
    if not hasattr(t, "data_ptr") or isinstance(t, np.ndarray):
        raise TypeError(f"{name}: expected a CUDA torch tensor, got {type(t).__name__}")
    if not t.is_cuda:
        raise ValueError(f"{name}: tensor is on {t.device}, the library needs device memory")
    if device is not None and t.device.index != device:
        raise ValueError(f"{name}: tensor is on {t.device}, the graph lives on cuda:{device}")
    if t.dtype != torch_float32():
        raise TypeError(f"{name}: dtype {t.dtype}, expected torch.float32")
    if not t.is_contiguous():
        raise ValueError(f"{name}: tensor is not contiguous")
    if t.numel() < numel:
        raise ValueError(f"{name}: {t.numel()} values, the call needs {numel}")
    return t.data_ptr()


def torch_float32():
    import torch
    return torch.float32


class Workspace:
    """xmgn_workspace_create / processor_fwd / processor_bwd for one GPU."""

    def __init__(self, graph, cfg, infer=False):
        """infer=True: xmgn_workspace_create_infer (forward only, no checkpoints)."""
        self.graph, self.cfg, self.infer = graph, cfg, infer
        h = _vp()
        create = _lib.xmgn_workspace_create_infer if infer else _lib.xmgn_workspace_create
        _check(create(graph.handle, ctypes.byref(cfg), ctypes.byref(h)))
        self.handle = h
        self.n_params = param_count(cfg)
        self._info = {}

    def nbytes(self):
        return int(_lib.xmgn_workspace_bytes(self.handle))

    def _sizes(self, part):
        if part not in self._info:
            self._info[part] = self.graph.part_info(part)
        i = self._info[part]
        return i["n_owned"], i["n_local"], i["e_local"]

    def forward(self, part, params, h0, e0, h_out, stream=None):
        no, nl, el = self._sizes(part)
        H, dv = self.cfg.hidden, self.graph.device
        _check(_lib.xmgn_processor_fwd(self.handle, int(part), _dev_f32(params, "params", self.n_params, dv),
                                       _dev_f32(h0, "h0", nl * H, dv), _dev_f32(e0, "e0", el * H, dv),
                                       _dev_f32(h_out, "h_out", no * H, dv), _stream(stream)))

    def backward(self, part, params, grad_h_out, grad_params, grad_h0=None, grad_e0=None, stream=None):
        no, nl, el = self._sizes(part)
        H, dv = self.cfg.hidden, self.graph.device
        _check(_lib.xmgn_processor_bwd(self.handle, int(part), _dev_f32(params, "params", self.n_params, dv),
                                       _dev_f32(grad_h_out, "grad_h_out", no * H, dv),
                                       _dev_f32(grad_params, "grad_params", self.n_params, dv),
                                       _dev_f32(grad_h0, "grad_h0", nl * H, dv),
                                       _dev_f32(grad_e0, "grad_e0", el * H, dv), _stream(stream)))

    def model_forward(self, part, params, io_params, pos, nrm, stats, pred, targets=None, n_global=0, loss=None,
                      stream=None):
        """xmgn_model_fwd: encoders -> processor -> decoder (-> owned-row MSE with targets)."""
        no, nl, el = self._sizes(part)
        dv = self.graph.device
        nio = io_param_count(self.cfg)
        _check(_lib.xmgn_model_fwd(self.handle, int(part), _dev_f32(params, "params", self.n_params, dv),
                                   _dev_f32(io_params, "io_params", nio, dv), _dev_f32(pos, "pos", nl * 3, dv),
                                   _dev_f32(nrm, "nrm", nl * 3, dv), _dev_f32(stats, "stats", IO_NSTATS, dv),
                                   _dev_f32(targets, "targets", no * IO_DOUT, dv), int(n_global),
                                   _dev_f32(pred, "pred", no * IO_DOUT, dv), _dev_f32(loss, "loss", 1, dv),
                                   _stream(stream)))

    def model_backward(self, part, params, io_params, grad_params, grad_io, stream=None):
        dv = self.graph.device
        nio = io_param_count(self.cfg)
        _check(_lib.xmgn_model_bwd(self.handle, int(part), _dev_f32(params, "params", self.n_params, dv),
                                   _dev_f32(io_params, "io_params", nio, dv),
                                   _dev_f32(grad_params, "grad_params", self.n_params, dv),
                                   _dev_f32(grad_io, "grad_io", nio, dv), _stream(stream)))

    def close(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.xmgn_workspace_free(self.handle)
        self.handle = None

    def __del__(self):
        self.close()


def check_finite(t, stream=None):
    _check(_lib.xmgn_check_finite(_dev_f32(t, "check_finite", t.numel()), t.numel(), _stream(stream)))


class Comm:
    """NCCL communicator for xmgn_grad_reduce (one per process / GPU)."""

    @staticmethod
    def unique_id():
        buf = ctypes.create_string_buffer(128)
        _check(_lib.xmgn_comm_unique_id(buf))
        return buf.raw

    def __init__(self, uid, nranks, rank, device):
        h = _vp()
        _check(_lib.xmgn_comm_init(bytes(uid), int(nranks), int(rank), int(device), ctypes.byref(h)))
        self.handle = h

    def grad_reduce(self, grad, stream=None):
        _check(_lib.xmgn_grad_reduce(self.handle, _dev_f32(grad, "grad", grad.numel()), grad.numel(),
                                     _stream(stream)))

    def gather_rows(self, send, recv=None, recv_rows=None, stream=None):
        """Rank 0 receives every rank's rows (send: [rows, W] CUDA float32) into recv in rank
        order; recv_rows: per-rank row counts (rank 0 only)."""
        W = send.shape[1] if send.dim() == 2 else 1
        rr = None
        if recv_rows is not None:
            rr = np.ascontiguousarray(recv_rows, dtype=np.int64)
            need = int(rr.sum()) * W
        _check(_lib.xmgn_gather_rows(self.handle, _dev_f32(send, "send", send.numel()), send.shape[0], W,
                                     _dev_f32(recv, "recv", need) if recv is not None else None,
                                     rr.ctypes.data if rr is not None else None, _stream(stream)))

    def close(self):
        if getattr(self, "handle", None):
            _lib.xmgn_comm_destroy(self.handle)
            self.handle = None


def scatter_rows(src, idx, dst, stream=None):
    """dst[idx[i]] = src[i] (rows; src/dst CUDA float32 2-D, idx CUDA int64)."""
    import torch
    n, W = src.shape
    if idx.dtype != torch.int64 or not idx.is_cuda or not idx.is_contiguous() or idx.numel() < n:
        raise TypeError("scatter_rows: idx must be a contiguous CUDA int64 tensor of >= n entries")
    if dst.dim() != 2 or dst.shape[1] != W:
        raise ValueError(f"scatter_rows: dst shape {tuple(dst.shape)} vs rows of width {W}")
    _check(_lib.xmgn_scatter_rows(_dev_f32(src, "src", n * W), idx.data_ptr(), n, W,
                                  _dev_f32(dst, "dst", dst.numel()), _stream(stream)))


class Adam:
    """xmgn_adam_step: global-norm clip + Adam + cosine LR on a flat FP32 parameter vector
    (PAPER.md:234 defaults: 1e-3 -> 1e-6, clip 32, betas 0.9 / 0.999, eps 1e-8)."""

    def __init__(self, n, total_steps, device=0, lr_max=1e-3, lr_min=1e-6, beta1=0.9, beta2=0.999, eps=1e-8,
                 clip=32.0):
        import torch
        self.cfg = AdamCfg(lr_max, lr_min, int(total_steps), beta1, beta2, eps, clip)
        self.m = torch.zeros(n, device=f"cuda:{device}")
        self.v = torch.zeros(n, device=f"cuda:{device}")
        self.norm = torch.zeros(1, device=f"cuda:{device}")
        self.t = 0

    def lr(self, step=None):
        return float(_lib.xmgn_cosine_lr(ctypes.byref(self.cfg), self.t if step is None else int(step)))

    def step(self, params, grad, grad_scale=1.0, stream=None):
        n = params.numel()
        _check(_lib.xmgn_adam_step(ctypes.byref(self.cfg), self.t, _dev_f32(params, "params", n),
                                   _dev_f32(grad, "grad", n), _dev_f32(self.m, "m", n), _dev_f32(self.v, "v", n), n,
                                   float(grad_scale), self.norm.data_ptr(), _stream(stream)))
        self.t += 1


def launch_count():
    return int(_lib.xmgn_launch_count())


def profile_enable(on=True):
    _check(_lib.xmgn_profile_enable(int(on)))


def profile_collect():
    """{scope name: (total ms, launches)} since the last collect."""
    buf = ctypes.create_string_buffer(4096)
    ms = (ctypes.c_double * 64)()
    cnt = (ctypes.c_longlong * 64)()
    n = _i32()
    _check(_lib.xmgn_profile_collect(buf, 4096, ms, cnt, 64, ctypes.byref(n)))
    names = buf.value.decode().split("\n")
    return {names[i]: (ms[i], int(cnt[i])) for i in range(n.value)}


def selftest_gemm(A, B, C, a_mn_major, b_mn_major, M, N, K, stream=None):
    _check(_lib.xmgn_selftest_gemm(M, N, K, int(a_mn_major), int(b_mn_major), _ptr(A), _ptr(B), _ptr(C),
                                   _stream(stream)))
