"""paper_2502_05370_b200 -- B200-native fMoE expert-map search (arXiv 2502.05370).

Thin ctypes binding over the C ABI in ``include/fmoe.h`` (libfmoe_b200.so,
sm_100a).  The functions below have the ABI's names and only marshal
arguments: every step of the path runs in the library's CUDA kernels.  Arrays
are torch tensors (CUDA tensors on the store's device, or CPU tensors -- the
library then stages them and synchronises).  PyTorch is used only for memory,
streams and process groups.  There is no CPU fallback: importing this package
without the built library raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libfmoe_b200.so")

FMOE_F32, FMOE_BF16 = 0, 1
FMOE_MAX_K = 64
FMOE_MAX_E = 64
_STATUS = {0: "ok", 1: "invalid argument", 2: "unsupported shape", 3: "out of device memory",
           4: "CUDA error", 5: "unsupported"}


class FmoeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"fmoe status {status} ({_STATUS.get(status, '?')}): {msg}")
        self.status = status


class fmoe_store_config(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int32), ("E", ctypes.c_int32), ("K", ctypes.c_int32), ("D", ctypes.c_int32),
                ("d", ctypes.c_int32), ("dtype", ctypes.c_int32), ("capacity", ctypes.c_int64),
                ("id_offset", ctypes.c_int64)]


# fmoe_allgather_fn (HOST transport of a sharded store): (send, recv, bytes, user) -> 0 on success
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)
FMOE_TRANSPORT_NCCL, FMOE_TRANSPORT_HOST = 0, 1


class fmoe_dist_config(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("transport", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("allgather", ALLGATHER_FN), ("allgather_user", ctypes.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2502_05370_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, F = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
    sig = {
        "fmoe_store_create": (I32, [ctypes.POINTER(fmoe_store_config), ctypes.c_int, ctypes.POINTER(P)]),
        "fmoe_store_create_sharded": (I32, [ctypes.POINTER(fmoe_store_config), ctypes.POINTER(fmoe_dist_config),
                                            ctypes.c_int, ctypes.POINTER(P)]),
        "fmoe_get_nccl_unique_id": (I32, [P]),
        "fmoe_store_destroy": (None, [P]),
        "fmoe_store_size": (I32, [P, ctypes.POINTER(I64)]),
        "fmoe_store_get_config": (I32, [P, ctypes.POINTER(fmoe_store_config)]),
        "fmoe_store_insert": (I32, [P, I64, P, P, P, P, P]),
        "fmoe_store_read": (I32, [P, I64, I64, P, P, P]),
        "fmoe_store_write": (I32, [P, I64, P, P, P, P]),
        "fmoe_store_insert_cos": (I32, [P, I64, P, P, P, I64, P, P, P]),
        "fmoe_search_semantic_cos": (I32, [P, I64, P, I32, P, P, P, I64, P]),
        "fmoe_resolve_victims": (I32, [I64, I32, P, P, ctypes.c_int, P]),
        "fmoe_search_semantic": (I32, [P, I64, P, I32, P, P, P]),
        "fmoe_search_trajectory": (I32, [P, I64, P, I32, I32, P, P, P]),
        "fmoe_search_blend": (I32, [P, I64, P, P, I32, F, I32, P, P, P]),
        "fmoe_search_blend_cos": (I32, [P, I64, P, I64, P, I32, F, I32, P, P, P]),
        "fmoe_select_experts": (I32, [P, I64, P, P, F, I32, I32, P, P, P]),
        "fmoe_traj_session_create": (I32, [P, I64, ctypes.POINTER(P)]),
        "fmoe_traj_session_step": (I32, [P, P, I32, P, P, P]),
        "fmoe_traj_session_step_select": (I32, [P, P, I32, P, P, F, I32, I32, P, P, P]),
        "fmoe_traj_session_sweep": (I32, [P, P, I32, P, P, F, I32, P, P, P, P, P]),
        "fmoe_traj_session_reset": (I32, [P]),
        "fmoe_traj_session_abandoned": (I32, [P, ctypes.POINTER(I32)]),
        "fmoe_traj_session_destroy": (None, [P]),
        "fmoe_topk_merge": (I32, [I64, I32, I32, P, P, I32, P, P, ctypes.c_int, P]),
        "fmoe_prefetch_plan": (I32, [P, I64, P, P, F, I32, I32, I32, I32, P, P, P, P, P]),
        "fmoe_eviction_order": (I32, [I64, P, P, F, P, P, ctypes.c_int, P]),
        "fmoe_prefetch_issue": (I32, [P, I64, P, P, F, I32, I32, I32, I32, P, P, I64, P, P, P, P, P, P]),
        "fmoe_expert_hits": (I32, [I64, I32, I32, I32, P, P, P, P, ctypes.c_int, P]),
        "fmoe_status_string": (ctypes.c_char_p, [I32]),
        "fmoe_last_error": (ctypes.c_char_p, []),
        "fmoe_kernel_launch_count": (I64, []),
        "fmoe_set_host_sync": (I32, [I32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()
ABI_SYMBOLS = ("fmoe_store_create", "fmoe_store_create_sharded", "fmoe_get_nccl_unique_id", "fmoe_store_destroy", "fmoe_store_size", "fmoe_store_get_config",
               "fmoe_store_insert", "fmoe_store_insert_cos", "fmoe_search_semantic_cos", "fmoe_store_read",
               "fmoe_store_write", "fmoe_resolve_victims", "fmoe_search_semantic", "fmoe_search_trajectory",
               "fmoe_search_blend", "fmoe_search_blend_cos", "fmoe_select_experts", "fmoe_traj_session_create", "fmoe_traj_session_step",
               "fmoe_traj_session_step_select", "fmoe_traj_session_sweep",
               "fmoe_traj_session_reset", "fmoe_traj_session_abandoned", "fmoe_traj_session_destroy", "fmoe_topk_merge",
               "fmoe_prefetch_plan", "fmoe_prefetch_issue", "fmoe_eviction_order", "fmoe_expert_hits", "fmoe_status_string",
               "fmoe_last_error", "fmoe_kernel_launch_count", "fmoe_set_host_sync")


def _check(st: int):
    if st != 0:
        raise FmoeError(st, _lib.fmoe_last_error().decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        if torch.cuda.is_available():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        return None
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _f32(t):
    assert t.dtype == torch.float32 and t.is_contiguous(), "fp32 contiguous tensor expected"
    return t


def kernel_launch_count() -> int:
    return int(_lib.fmoe_kernel_launch_count())


# ------------------------------------------------------------------ ABI-named functions
def fmoe_store_create(L, E, K, D, d, capacity, dtype="bf16", device=0, id_offset=0):
    cfg = fmoe_store_config(L, E, K, D, d, FMOE_BF16 if dtype == "bf16" else FMOE_F32, capacity, id_offset)
    h = ctypes.c_void_p()
    _check(_lib.fmoe_store_create(ctypes.byref(cfg), int(device), ctypes.byref(h)))
    return h


def fmoe_get_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.fmoe_get_nccl_unique_id(buf))
    return buf.raw


def fmoe_store_create_sharded(L, E, K, D, d, capacity_total, dtype="bf16", device=0, rank=0, world=1,
                              transport="nccl", nccl_unique_id=None, host_allgather=None):
    """This rank's shard of a store of capacity_total global slots (collective).
    transport "nccl": nccl_unique_id = the 128 bytes of fmoe_get_nccl_unique_id (same on
    every rank); "host": host_allgather = an object whose .cfn is an ALLGATHER_FN."""
    cfg = fmoe_store_config(L, E, K, D, d, FMOE_BF16 if dtype == "bf16" else FMOE_F32, capacity_total, 0)
    uid = ctypes.create_string_buffer(nccl_unique_id, 128) if nccl_unique_id is not None else None
    dc = fmoe_dist_config(rank, world, FMOE_TRANSPORT_NCCL if transport == "nccl" else FMOE_TRANSPORT_HOST,
                          ctypes.cast(uid, ctypes.c_void_p) if uid is not None else None,
                          host_allgather.cfn if host_allgather is not None else ALLGATHER_FN(), None)
    h = ctypes.c_void_p()
    _check(_lib.fmoe_store_create_sharded(ctypes.byref(cfg), ctypes.byref(dc), int(device), ctypes.byref(h)))
    return h


def fmoe_store_destroy(h):
    _lib.fmoe_store_destroy(h)


def fmoe_store_size(h) -> int:
    n = ctypes.c_int64()
    _check(_lib.fmoe_store_size(h, ctypes.byref(n)))
    return n.value


def fmoe_store_insert(h, emb, maps, out_slot=None, out_replaced=None, stream=None):
    _check(_lib.fmoe_store_insert(h, emb.shape[0], _ptr(_f32(emb)), _ptr(_f32(maps)), _ptr(out_slot),
                                  _ptr(out_replaced), _stream(stream)))


def fmoe_store_insert_cos(h, emb, maps, sem_cos, cos_stride, out_slot=None, out_replaced=None, stream=None):
    _check(_lib.fmoe_store_insert_cos(h, emb.shape[0], _ptr(_f32(emb)), _ptr(_f32(maps)),
                                      _ptr(None if sem_cos is None else _f32(sem_cos)), cos_stride,
                                      _ptr(out_slot), _ptr(out_replaced), _stream(stream)))


def fmoe_search_semantic_cos(h, q_emb, k, out_score, out_id, out_cos, cos_stride, stream=None):
    _check(_lib.fmoe_search_semantic_cos(h, q_emb.shape[0], _ptr(_f32(q_emb)), k, _ptr(out_score), _ptr(out_id),
                                         _ptr(out_cos), cos_stride, _stream(stream)))


def fmoe_store_write(h, emb, maps, slot, stream=None):
    _check(_lib.fmoe_store_write(h, emb.shape[0], _ptr(_f32(emb)), _ptr(_f32(maps)), _ptr(slot), _stream(stream)))


def fmoe_resolve_victims(ids, out_victim, device=0, stream=None):
    B, k = ids.shape
    _check(_lib.fmoe_resolve_victims(B, k, _ptr(ids), _ptr(out_victim), int(device), _stream(stream)))


def fmoe_store_read(h, slot_begin, count, out_emb=None, out_maps=None, stream=None):
    _check(_lib.fmoe_store_read(h, slot_begin, count, _ptr(out_emb), _ptr(out_maps), _stream(stream)))


def fmoe_search_semantic(h, q_emb, k, out_score, out_id, stream=None):
    _check(_lib.fmoe_search_semantic(h, q_emb.shape[0], _ptr(_f32(q_emb)), k, _ptr(out_score), _ptr(out_id),
                                     _stream(stream)))


def fmoe_search_trajectory(h, q_prefix, ell, k, out_score, out_id, stream=None):
    _check(_lib.fmoe_search_trajectory(h, q_prefix.shape[0], _ptr(_f32(q_prefix)), ell, k, _ptr(out_score),
                                       _ptr(out_id), _stream(stream)))


def fmoe_search_blend(h, q_emb, q_prefix, ell, w_sem, k, out_score, out_id, stream=None):
    _check(_lib.fmoe_search_blend(h, q_emb.shape[0], _ptr(_f32(q_emb)), _ptr(_f32(q_prefix)), ell, w_sem, k,
                                  _ptr(out_score), _ptr(out_id), _stream(stream)))


def fmoe_search_blend_cos(h, sem_cos, cos_stride, q_prefix, ell, w_sem, k, out_score, out_id, stream=None):
    _check(_lib.fmoe_search_blend_cos(h, q_prefix.shape[0], _ptr(_f32(sem_cos)), cos_stride, _ptr(_f32(q_prefix)), ell, w_sem, k,
                                      _ptr(out_score), _ptr(out_id), _stream(stream)))


def fmoe_select_experts(h, map_id, score, delta, layer_begin, layer_end, out_mask, out_count, stream=None):
    _check(_lib.fmoe_select_experts(h, map_id.shape[0], _ptr(map_id), _ptr(score), delta, layer_begin, layer_end,
                                    _ptr(out_mask), _ptr(out_count), _stream(stream)))


def fmoe_prefetch_plan(h, map_id, score, delta, l_now, layer_begin, layer_end, max_jobs, out_layer, out_expert,
                       out_priority, out_njobs, stream=None):
    _check(_lib.fmoe_prefetch_plan(h, map_id.shape[0], _ptr(map_id), _ptr(score), delta, l_now, layer_begin, layer_end,
                                   max_jobs, _ptr(out_layer), _ptr(out_expert), _ptr(out_priority), _ptr(out_njobs),
                                   _stream(stream)))


def fmoe_prefetch_issue(h, map_id, score, delta, l_now, layer_begin, layer_end, max_jobs, host_expert_ptrs,
                        dev_expert_ptrs, expert_bytes, resident_mask=None, wait_flag=None, copy_stream=None):
    """Issue the expert copies of the prefetch plan (include/fmoe.h).  host_expert_ptrs /
    dev_expert_ptrs: sequences of L*E addresses (int); resident_mask: CPU int64 tensor [L]
    (updated in place) or None.  Returns (layers, experts, njobs) host tensors of the copies issued."""
    B = map_id.shape[0]
    n = len(host_expert_ptrs)
    hp = (ctypes.c_void_p * n)(*host_expert_ptrs)
    dp = (ctypes.c_void_p * n)(*dev_expert_ptrs)
    lay = torch.empty(B, max_jobs, dtype=torch.int32)
    exp = torch.empty(B, max_jobs, dtype=torch.int32)
    nj = torch.empty(B, dtype=torch.int32)
    _check(_lib.fmoe_prefetch_issue(h, B, _ptr(map_id), _ptr(score), delta, l_now, layer_begin, layer_end, max_jobs,
                                    hp, dp, int(expert_bytes), _ptr(resident_mask), _ptr(wait_flag),
                                    _stream(copy_stream), _ptr(lay), _ptr(exp), _ptr(nj)))
    return lay, exp, nj


def fmoe_eviction_order(p, freq, eps, out_priority, out_order, device=0, stream=None):
    _check(_lib.fmoe_eviction_order(p.shape[0], _ptr(p), _ptr(freq), eps, _ptr(out_priority), _ptr(out_order),
                                    int(device), _stream(stream)))


def fmoe_expert_hits(gate, prefetch_mask, K, out_hits, out_active=None, device=0, stream=None):
    """gate [B][T][E] fp32, prefetch_mask [B][T] (u)int64 -> out_hits [B][T] int32 (+ out_active)."""
    B, T, E = gate.shape
    _check(_lib.fmoe_expert_hits(B, T, E, K, _ptr(gate), _ptr(prefetch_mask), _ptr(out_active), _ptr(out_hits),
                                 int(device), _stream(stream)))


def fmoe_traj_session_create(h, B):
    s = ctypes.c_void_p()
    _check(_lib.fmoe_traj_session_create(h, B, ctypes.byref(s)))
    return s


def fmoe_traj_session_step(s, q_layer, k, out_score, out_id, stream=None):
    _check(_lib.fmoe_traj_session_step(s, _ptr(_f32(q_layer)), k, _ptr(out_score), _ptr(out_id), _stream(stream)))


def fmoe_traj_session_step_select(s, q_layer, k, out_score, out_id, delta, layer_begin, layer_end, out_mask,
                                  out_count, stream=None):
    _check(_lib.fmoe_traj_session_step_select(s, _ptr(_f32(q_layer)), k, _ptr(out_score), _ptr(out_id), delta,
                                              layer_begin, layer_end, _ptr(out_mask), _ptr(out_count),
                                              _stream(stream)))


def fmoe_traj_session_sweep(s, q_layers, out_score, out_id, delta=-1.0, sel_d=-1, out_mask=None, out_count=None,
                            layer_ready=None, guidance_ready=None, stream=None):
    """q_layers [n_steps][B][E] -> out_score/out_id [n_steps][B] (+ selection masks/counts)."""
    _check(_lib.fmoe_traj_session_sweep(s, _ptr(_f32(q_layers)), q_layers.shape[0], _ptr(out_score), _ptr(out_id), delta,
                                        sel_d, _ptr(out_mask), _ptr(out_count), _ptr(layer_ready),
                                        _ptr(guidance_ready), _stream(stream)))


def fmoe_set_host_sync(enable):
    """Process-wide: whether calls with host outputs synchronise (see include/fmoe.h).
    Returns the previous setting."""
    return int(_lib.fmoe_set_host_sync(1 if enable else 0))


def fmoe_traj_session_reset(s):
    _check(_lib.fmoe_traj_session_reset(s))


def fmoe_traj_session_abandoned(s) -> bool:
    """Whether a sweep of the session was abandoned (layer_ready timeout) since the last reset;
    read after synchronising the sweep's stream."""
    v = ctypes.c_int32()
    _check(_lib.fmoe_traj_session_abandoned(s, ctypes.byref(v)))
    return bool(v.value)


def fmoe_traj_session_destroy(s):
    _lib.fmoe_traj_session_destroy(s)


def fmoe_topk_merge(scores, ids, k, out_score, out_id, device=0, stream=None):
    n_lists, B, k_in = scores.shape
    _check(_lib.fmoe_topk_merge(B, n_lists, k_in, _ptr(scores), _ptr(ids), k, _ptr(out_score), _ptr(out_id),
                                int(device), _stream(stream)))


# ------------------------------------------------------------------ convenience object
class ExpertMapStore:
    """Owning wrapper: allocates outputs as torch tensors on the store's device."""

    def __init__(self, L, E, K, D, d=3, capacity=1024, dtype="bf16", device=0, id_offset=0):
        self.L, self.E, self.K, self.D, self.d = L, E, K, D, d
        self.capacity, self.dtype, self.id_offset = capacity, dtype, id_offset
        self.device = torch.device("cuda", device)
        self._h = fmoe_store_create(L, E, K, D, d, capacity, dtype, device, id_offset)

    def close(self):
        if self._h is not None:
            fmoe_store_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __len__(self):
        return fmoe_store_size(self._h)

    def insert(self, emb, maps, stream=None):
        B = emb.shape[0]
        slot = torch.empty(B, dtype=torch.int64, device=self.device)
        rep = torch.empty(B, dtype=torch.int64, device=self.device)
        fmoe_store_insert(self._h, emb, maps, slot, rep, stream)
        return slot, rep

    def read(self, slot_begin=0, count=None):
        count = len(self) - slot_begin if count is None else count
        e = torch.empty(count, self.D, device=self.device)
        m = torch.empty(count, self.L, self.E, device=self.device)
        fmoe_store_read(self._h, slot_begin, count, e, m)
        return e, m

    def _out(self, B, k):
        return (torch.empty(B, k, dtype=torch.float32, device=self.device),
                torch.empty(B, k, dtype=torch.int64, device=self.device))

    def search_semantic(self, q_emb, k=1, stream=None):
        s, i = self._out(q_emb.shape[0], k)
        fmoe_search_semantic(self._h, q_emb, k, s, i, stream)
        return s, i

    def search_trajectory(self, q_prefix, ell, k=1, stream=None):
        q_prefix = q_prefix[:, :ell].contiguous()
        s, i = self._out(q_prefix.shape[0], k)
        fmoe_search_trajectory(self._h, q_prefix, ell, k, s, i, stream)
        return s, i

    def search_blend(self, q_emb, q_prefix, ell, w_sem=-1.0, k=1, stream=None):
        q_prefix = q_prefix[:, :ell].contiguous()
        s, i = self._out(q_emb.shape[0], k)
        fmoe_search_blend(self._h, q_emb, q_prefix, ell, w_sem, k, s, i, stream)
        return s, i

    def trajectory_session(self, B):
        return TrajectorySession(self, B)

    def select_experts(self, map_id, score, delta=-1.0, layer_begin=0, layer_end=None, stream=None):
        layer_end = self.L if layer_end is None else layer_end
        B, T = map_id.shape[0], layer_end - layer_begin
        mask = torch.empty(B, T, dtype=torch.int64, device=self.device)   # uint64 bit pattern
        cnt = torch.empty(B, T, dtype=torch.int32, device=self.device)
        fmoe_select_experts(self._h, map_id.contiguous(), None if score is None else score.contiguous(), delta,
                            layer_begin, layer_end, mask, cnt, stream)
        return mask, cnt


def expert_hits(gate, prefetch_mask, K, stream=None):
    """Hits of prefetch guidance: gate [B][T][E] fp32, prefetch_mask [B][T] int64 (uint64 bits)
    -> (hits [B][T] int32, activated masks [B][T] int64)."""
    B, T, _ = gate.shape
    hits = torch.empty(B, T, dtype=torch.int32, device=gate.device)
    act = torch.empty(B, T, dtype=torch.int64, device=gate.device)
    fmoe_expert_hits(gate.contiguous(), prefetch_mask.contiguous(), K, hits, act,
                     gate.device.index or 0, stream)
    return hits, act


class TrajectorySession:
    """Incremental trajectory search: step() consumes the next layer of each query."""

    def __init__(self, store, B):
        self.store, self.B = store, B
        self._s = fmoe_traj_session_create(store._h, B)

    def step(self, q_layer, k=1, stream=None):
        s = torch.empty(self.B, k, dtype=torch.float32, device=self.store.device)
        i = torch.empty(self.B, k, dtype=torch.int64, device=self.store.device)
        fmoe_traj_session_step(self._s, q_layer.contiguous(), k, s, i, stream)
        return s, i

    def step_select(self, q_layer, k, delta, layer_begin, layer_end, stream=None):
        """step() followed by select_experts() on each query's top-1, in one call."""
        dev = self.store.device
        s = torch.empty(self.B, k, dtype=torch.float32, device=dev)
        i = torch.empty(self.B, k, dtype=torch.int64, device=dev)
        T = layer_end - layer_begin
        mask = torch.empty(self.B, T, dtype=torch.int64, device=dev)   # uint64 bit pattern
        cnt = torch.empty(self.B, T, dtype=torch.int32, device=dev)
        fmoe_traj_session_step_select(self._s, q_layer.contiguous(), k, s, i, delta, layer_begin, layer_end, mask,
                                      cnt, stream)
        return s, i, mask, cnt

    def sweep(self, q_layers, delta=-1.0, sel_d=None, layer_ready=None, guidance_ready=None, stream=None):
        """n = q_layers.shape[0] steps in one call (k = 1): q_layers [n][B][E] -> scores, ids [n][B] and
        the selection masks / counts [n][B] of target layer (consumed layer + sel_d) (None: no selection)."""
        dev = self.store.device
        n = q_layers.shape[0]
        s = torch.empty(n, self.B, dtype=torch.float32, device=dev)
        i = torch.empty(n, self.B, dtype=torch.int64, device=dev)
        mask = cnt = None
        if sel_d is not None:
            mask = torch.empty(n, self.B, dtype=torch.int64, device=dev)
            cnt = torch.empty(n, self.B, dtype=torch.int32, device=dev)
        fmoe_traj_session_sweep(self._s, q_layers.contiguous(), s, i, delta, -1 if sel_d is None else sel_d, mask,
                                cnt, layer_ready, guidance_ready, stream)
        return s, i, mask, cnt

    def reset(self):
        fmoe_traj_session_reset(self._s)

    def close(self):
        if self._s is not None:
            fmoe_traj_session_destroy(self._s)
            self._s = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
