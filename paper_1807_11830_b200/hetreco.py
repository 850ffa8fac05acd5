"""Python mirror of the hetreco operator API over the C-ABI (include/hetreco_b200.h).

This is the ctypes binding a maintainer would add on the reference side: the
same names, argument meaning and error types as the reference's C++ API
(include/hetreco/{device,ndarray,layout,session,process}.hpp), backed by
libhetreco_b200.so.  Arrays are numpy arrays in Fortran order whose ``shape``
equals the reference ``dims`` (column-major, fastest dim first,
ndarray.hpp:61-67).  There is no CPU fallback: if the shared library is
missing the import fails, and without a GPU ``ComputeSession`` raises
``NoMatchingDevice``.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import weakref
from typing import Iterable, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhetreco_b200.so")

# ---------------------------------------------------------------------------
# errors (include/hetreco/errors.hpp; codes = hetreco::ErrorCode)
# ---------------------------------------------------------------------------


class HetrecoError(RuntimeError):
    code = 1


_ERROR_NAMES = ["Ok", "Error", "InvalidFilter", "NoMatchingDevice", "InvalidArgument", "EmptyData", "Overflow",
                "MalformedHeader", "AllocationFailure", "UnknownHandle", "DeviceError", "CompileError",
                "DuplicateKernel", "UnsupportedSource", "UnknownKernel", "InvalidParams", "ShapeMismatch",
                "AlreadyInitialized", "NotInitialized", "ChainMismatch", "ChainStageError",
                "UnsupportedElementType", "MalformedFile", "UnsupportedFeature", "IoError", "SizeMismatch",
                "MalformedSidecar"]
ERRORS: dict[int, type] = {1: HetrecoError}
for _code, _name in enumerate(_ERROR_NAMES):
    if _code >= 2:
        ERRORS[_code] = type(_name, (HetrecoError,), {"code": _code})
        globals()[_name] = ERRORS[_code]
Error = HetrecoError

# ---------------------------------------------------------------------------
# library loading
# ---------------------------------------------------------------------------

_lib = None


class _DeviceDesc(C.Structure):
    _fields_ = [("backend_id", C.c_char * 32), ("device_index", C.c_uint32), ("device_type", C.c_int32),
                ("vendor", C.c_char * 32), ("name", C.c_char * 128), ("api_version", C.c_char * 16),
                ("global_memory_bytes", C.c_uint64), ("base_alignment_bytes", C.c_uint64),
                ("supports_source_kernels", C.c_int32)]


class _Handle(C.Structure):
    _fields_ = [("session_uid", C.c_uint64), ("id", C.c_uint64)]


class _ArrayDesc(C.Structure):
    _fields_ = [("element_type", C.c_uint64), ("rank", C.c_uint32), ("_pad", C.c_uint32),
                ("dims", C.c_uint64 * 8), ("offset_bytes", C.c_uint64), ("host", C.c_void_p)]


EXPORTED = [
    "hetreco_last_error", "hetreco_version", "hetreco_enumerate_devices", "hetreco_select_device",
    "hetreco_select_from", "hetreco_cuda_device_count", "hetreco_cuda_backend_create",
    "hetreco_cuda_backend_destroy", "hetreco_cuda_backend_device", "hetreco_cuda_allocate", "hetreco_cuda_release",
    "hetreco_cuda_upload", "hetreco_cuda_download", "hetreco_cuda_copy", "hetreco_cuda_kernel_count",
    "hetreco_cuda_kernel_name", "hetreco_cuda_execute", "hetreco_cuda_synchronize", "hetreco_host_alloc",
    "hetreco_host_free", "hetreco_session_create", "hetreco_session_create_on", "hetreco_session_destroy",
    "hetreco_session_device", "hetreco_register_data", "hetreco_allocate_data", "hetreco_session_layout",
    "hetreco_fetch_data", "hetreco_release_data", "hetreco_fetch_header_bytes", "hetreco_copy_array",
    "hetreco_load_builtin_kernels", "hetreco_kernel_names", "hetreco_load_kernels", "hetreco_launch_kernel",
    "hetreco_synchronize", "hetreco_counters", "hetreco_reset_counters", "hetreco_live_data_count",
    "hetreco_params_create", "hetreco_params_destroy", "hetreco_params_set_bool", "hetreco_params_set_int",
    "hetreco_params_set_real", "hetreco_params_set_string", "hetreco_process_create", "hetreco_chain_create",
    "hetreco_process_destroy", "hetreco_process_set_input", "hetreco_process_set_output", "hetreco_process_init",
    "hetreco_process_launch", "hetreco_process_state", "hetreco_process_stats", "hetreco_chain_stage",
    "hetreco_stream_create", "hetreco_stream_run", "hetreco_stream_destroy", "hetreco_pack_layout",
    "hetreco_parse_layout_header", "hetreco_filter_describe", "hetreco_process_profile",
    "hetreco_session_timer_start", "hetreco_session_timer_stop",
    "hetreco_mat_read", "hetreco_mat_parse", "hetreco_image_read", "hetreco_raw_read", "hetreco_mat_count",
    "hetreco_mat_variable", "hetreco_mat_free", "hetreco_mat_write", "hetreco_image_write", "hetreco_raw_write",
    "hetreco_gen_phantom", "hetreco_phantom_blobs", "hetreco_nvrtc_compile_check", "hetreco_nvrtc_available",
    "hetreco_cuda_supports_source", "hetreco_cuda_compile", "hetreco_cuda_execute_unit",
    "hetreco_device_numa_node", "hetreco_bind_numa_node", "hetreco_parse_cpulist",
    "hetreco_frame_slab", "hetreco_multi_create", "hetreco_multi_run", "hetreco_multi_slab",
    "hetreco_multi_device_count", "hetreco_multi_destroy",
]


def lib():
    """Load libhetreco_b200.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1807_11830_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u64, i32, pc = C.c_void_p, C.c_uint64, C.c_int, C.c_char_p
    H = _Handle
    sig = {
        "hetreco_last_error": ([], pc), "hetreco_version": ([], pc),
        "hetreco_enumerate_devices": ([vp, i32, vp], i32), "hetreco_select_device": ([pc, vp], i32),
        "hetreco_select_from": ([vp, i32, pc, vp], i32), "hetreco_filter_describe": ([pc, vp, u64], i32),
        "hetreco_cuda_device_count": ([vp], i32), "hetreco_cuda_backend_create": ([i32, u64, vp], i32),
        "hetreco_cuda_backend_destroy": ([vp], i32), "hetreco_cuda_backend_device": ([vp, vp], i32),
        "hetreco_cuda_allocate": ([vp, u64, vp], i32), "hetreco_cuda_release": ([vp, u64], i32),
        "hetreco_cuda_upload": ([vp, u64, u64, vp, u64], i32), "hetreco_cuda_download": ([vp, u64, u64, vp, u64], i32),
        "hetreco_cuda_copy": ([vp, u64, u64, u64, u64, u64], i32), "hetreco_cuda_kernel_count": ([vp], i32),
        "hetreco_cuda_kernel_name": ([i32], pc),
        "hetreco_cuda_execute": ([vp, pc, u64, u64, u64, u64, vp, u64, u64], i32),
        "hetreco_cuda_synchronize": ([vp], i32), "hetreco_host_alloc": ([u64, vp], i32),
        "hetreco_host_free": ([vp], i32), "hetreco_session_create": ([pc, vp], i32),
        "hetreco_session_create_on": ([pc, vp], i32), "hetreco_session_destroy": ([vp], i32),
        "hetreco_session_device": ([vp, vp], i32), "hetreco_register_data": ([vp, i32, i32, vp, vp], i32),
        "hetreco_allocate_data": ([vp, i32, i32, vp, vp], i32),
        "hetreco_session_layout": ([vp, H, vp, i32, vp, vp, vp], i32),
        "hetreco_fetch_data": ([vp, H, i32, vp], i32), "hetreco_release_data": ([vp, H], i32),
        "hetreco_fetch_header_bytes": ([vp, H, vp, u64, vp], i32),
        "hetreco_copy_array": ([vp, H, u64, H, u64], i32), "hetreco_load_builtin_kernels": ([vp], i32),
        "hetreco_kernel_names": ([vp, vp, u64], i32), "hetreco_load_kernels": ([vp, i32, vp, vp], i32),
        "hetreco_launch_kernel": ([vp, pc, H, H, vp, u64, u64], i32), "hetreco_synchronize": ([vp], i32),
        "hetreco_counters": ([vp, vp, vp], i32), "hetreco_reset_counters": ([vp], i32),
        "hetreco_live_data_count": ([vp, vp], i32), "hetreco_params_create": ([vp], i32),
        "hetreco_params_destroy": ([vp], i32), "hetreco_params_set_bool": ([vp, pc, i32], i32),
        "hetreco_params_set_int": ([vp, pc, C.c_int64], i32), "hetreco_params_set_real": ([vp, pc, C.c_double], i32),
        "hetreco_params_set_string": ([vp, pc, pc], i32), "hetreco_process_create": ([vp, pc, pc, vp], i32),
        "hetreco_chain_create": ([vp, pc, vp, i32, vp], i32), "hetreco_process_destroy": ([vp], i32),
        "hetreco_process_set_input": ([vp, H], i32), "hetreco_process_set_output": ([vp, H], i32),
        "hetreco_process_init": ([vp, vp], i32), "hetreco_process_launch": ([vp], i32),
        "hetreco_process_state": ([vp, vp], i32), "hetreco_process_stats": ([vp, vp, vp, vp, vp, vp], i32),
        "hetreco_chain_stage": ([vp, i32, vp], i32),
        "hetreco_process_profile": ([vp, i32, vp, i32, vp], i32),
        "hetreco_session_timer_start": ([vp], i32), "hetreco_session_timer_stop": ([vp, vp], i32),
        "hetreco_stream_create": ([vp, i32, u64, u64, u64, u64, vp, i32, vp], i32),
        "hetreco_stream_run": ([vp, vp, u64, vp], i32), "hetreco_stream_destroy": ([vp], i32),
        "hetreco_pack_layout": ([i32, vp, u64, vp, u64, vp], i32),
        "hetreco_parse_layout_header": ([vp, u64, vp, i32, vp, vp, vp], i32),
    }
    sig.update({
        "hetreco_mat_read": ([pc, i32, vp], i32), "hetreco_mat_parse": ([vp, u64, i32, vp], i32),
        "hetreco_image_read": ([pc, i32, vp], i32), "hetreco_raw_read": ([pc, pc, i32, vp], i32),
        "hetreco_mat_count": ([vp, vp], i32), "hetreco_mat_variable": ([vp, i32, vp, u64, vp], i32),
        "hetreco_mat_free": ([vp], i32), "hetreco_mat_write": ([pc, i32, vp, vp], i32),
        "hetreco_image_write": ([pc, vp], i32), "hetreco_raw_write": ([pc, pc, vp], i32),
        "hetreco_gen_phantom": ([vp, u64, u64, u64, u64, u64, vp, vp, vp], i32),
        "hetreco_phantom_blobs": ([u64, u64, u64, vp], i32),
        "hetreco_nvrtc_compile_check": ([pc, pc, vp, u64, vp, u64], i32), "hetreco_nvrtc_available": ([vp], i32),
        "hetreco_cuda_supports_source": ([vp, vp], i32), "hetreco_cuda_compile": ([vp, i32, vp, vp, vp, u64], i32),
        "hetreco_cuda_execute_unit": ([vp, pc, pc, u64, u64, u64, u64, vp, u64, u64], i32),
        "hetreco_device_numa_node": ([i32, vp], i32), "hetreco_bind_numa_node": ([i32, vp], i32),
        "hetreco_parse_cpulist": ([pc, vp, i32, vp], i32),
        "hetreco_frame_slab": ([u64, u64, u64, vp, vp], i32),
        "hetreco_multi_create": ([i32, vp, i32, u64, u64, u64, u64, vp, i32, i32, vp], i32),
        "hetreco_multi_run": ([vp, vp, u64, vp], i32), "hetreco_multi_slab": ([vp, i32, vp, vp, vp], i32),
        "hetreco_multi_device_count": ([vp, vp], i32), "hetreco_multi_destroy": ([vp], i32),
    })
    lenient = os.environ.get("HETRECO_LIB_LENIENT") == "1"  # A/B runs against older builds
    for name, (args, res) in sig.items():
        if lenient and not hasattr(L, name):
            continue
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _ck(rc: int):
    if rc != 0:
        msg = lib().hetreco_last_error().decode(errors="replace")
        raise ERRORS.get(rc, HetrecoError)(msg)


# ---------------------------------------------------------------------------
# element types, arrays, data (ndarray.hpp / layout.hpp)
# ---------------------------------------------------------------------------


class ElementType(enum.IntEnum):
    UInt8 = 1
    Int32 = 2
    Float32 = 3
    Complex64 = 4
    Float64 = 5
    Complex128 = 6


_NP = {ElementType.UInt8: np.uint8, ElementType.Int32: np.int32, ElementType.Float32: np.float32,
       ElementType.Complex64: np.complex64, ElementType.Float64: np.float64,
       ElementType.Complex128: np.complex128}
_ET = {np.dtype(v): k for k, v in _NP.items()}


def element_type_of(dtype) -> ElementType:
    try:
        return _ET[np.dtype(dtype)]
    except KeyError:
        raise UnsupportedElementType(f"dtype {dtype} has no hetreco ElementType") from None  # noqa: F821


def dtype_of(t: int):
    return _NP[ElementType(t)]


class DataKind(enum.IntEnum):
    XData = 0
    KData = 1
    Generic = 2


class Data:
    """Ordered heterogeneous arrays moved as one unit (ndarray.hpp:139-152)."""

    def __init__(self, arrays: Sequence[np.ndarray] = (), kind: DataKind = DataKind.Generic):
        self.arrays = [np.asfortranarray(a) for a in arrays]
        self.kind = DataKind(kind)

    def array_count(self) -> int:
        return len(self.arrays)

    def empty(self) -> bool:
        return not self.arrays

    def payload_byte_size(self) -> int:
        return sum(a.nbytes for a in self.arrays)


def _desc(shape, dtype, host=None) -> _ArrayDesc:
    d = _ArrayDesc()
    d.element_type = int(element_type_of(dtype))
    shape = tuple(shape) if len(shape) else (1,)
    d.rank = len(shape)
    for i, n in enumerate(shape[:8]):
        d.dims[i] = int(n)
    for i in range(len(shape), 8):
        d.dims[i] = 1
    d.host = host
    return d


def _descs(arrays: Sequence[np.ndarray]):
    arr = (_ArrayDesc * max(1, len(arrays)))()
    for i, a in enumerate(arrays):
        arr[i] = _desc(a.shape, a.dtype, a.ctypes.data)
    return arr


class LayoutRecord:
    def __init__(self, d: _ArrayDesc):
        self.element_type = ElementType(d.element_type)
        self.rank = int(d.rank)
        self.dims = [int(d.dims[i]) for i in range(8)]
        self.offset_bytes = int(d.offset_bytes)

    @property
    def shape(self):
        return tuple(self.dims[:self.rank])

    def byte_size(self) -> int:
        return int(np.prod(self.shape)) * np.dtype(dtype_of(self.element_type)).itemsize

    def __repr__(self):
        return f"LayoutRecord(off={self.offset_bytes}, {self.element_type.name}, {self.shape})"


class LayoutDescriptor:
    def __init__(self, records, total_bytes, alignment_bytes=None):
        self.records = records
        self.total_bytes = int(total_bytes)
        self.alignment_bytes = alignment_bytes

    def array_count(self):
        return len(self.records)


def pack_layout(arrays_or_shapes, alignment: int = 256):
    """pack() + serialize_layout_header() (layout.cpp:57-102).
    Returns (LayoutDescriptor, header u64 words)."""
    items = [(a.shape, a.dtype) if isinstance(a, np.ndarray) else a for a in arrays_or_shapes]
    n = len(items)
    descs = (_ArrayDesc * max(1, n))()
    for i, (shape, dt) in enumerate(items):
        descs[i] = _desc(shape, dt)
    words = np.zeros(1 + 11 * n, np.uint64)
    total = C.c_uint64()
    _ck(lib().hetreco_pack_layout(n, descs, alignment, words.ctypes.data, words.size, C.byref(total)))
    return LayoutDescriptor([LayoutRecord(descs[i]) for i in range(n)], total.value, alignment), words


def parse_layout_header(data: bytes) -> LayoutDescriptor:
    buf = np.frombuffer(bytes(data) or b"\0" * 8, np.uint8).copy()
    cap = max(1, len(data) // 88 + 1)
    out = (_ArrayDesc * cap)()
    n, align, total = C.c_int(), C.c_uint64(), C.c_uint64()
    _ck(lib().hetreco_parse_layout_header(buf.ctypes.data, len(data), out, cap, C.byref(n), C.byref(align),
                                          C.byref(total)))
    return LayoutDescriptor([LayoutRecord(out[i]) for i in range(n.value)], total.value, align.value)


# ---------------------------------------------------------------------------
# devices (device.hpp)
# ---------------------------------------------------------------------------


class DeviceType(enum.IntEnum):
    Cpu = 0
    Gpu = 1
    Accelerator = 2


class DeviceDescriptor:
    def __init__(self, d: _DeviceDesc):
        self.backend_id = d.backend_id.decode()
        self.device_index = int(d.device_index)
        self.device_type = DeviceType(d.device_type)
        self.vendor = d.vendor.decode()
        self.name = d.name.decode()
        self.api_version = d.api_version.decode()
        self.global_memory_bytes = int(d.global_memory_bytes)
        self.base_alignment_bytes = int(d.base_alignment_bytes)
        self.supports_source_kernels = bool(d.supports_source_kernels)

    def label(self):
        return f"{self.backend_id}:{self.name}"

    def _c(self) -> _DeviceDesc:
        d = _DeviceDesc()
        d.backend_id = self.backend_id.encode()[:31]
        d.device_index = self.device_index
        d.device_type = int(self.device_type)
        d.vendor = self.vendor.encode()[:31]
        d.name = self.name.encode()[:127]
        d.api_version = self.api_version.encode()[:15]
        d.global_memory_bytes = self.global_memory_bytes
        d.base_alignment_bytes = self.base_alignment_bytes
        d.supports_source_kernels = int(self.supports_source_kernels)
        return d

    @staticmethod
    def make(backend_id="x", device_type=DeviceType.Cpu, vendor="", name="", api_version="1.0",
             global_memory_bytes=1, base_alignment_bytes=256):
        d = _DeviceDesc()
        d.backend_id = backend_id.encode()
        d.device_type = int(device_type)
        d.vendor = vendor.encode()
        d.name = name.encode()
        d.api_version = api_version.encode()
        d.global_memory_bytes = global_memory_bytes
        d.base_alignment_bytes = base_alignment_bytes
        return DeviceDescriptor(d)

    def __repr__(self):
        return f"DeviceDescriptor({self.label()}, {self.device_type.name}, api={self.api_version})"


def enumerate_devices():
    cnt = C.c_int()
    _ck(lib().hetreco_enumerate_devices(None, 0, C.byref(cnt)))
    arr = (_DeviceDesc * max(1, cnt.value))()
    _ck(lib().hetreco_enumerate_devices(arr, cnt.value, C.byref(cnt)))
    return [DeviceDescriptor(arr[i]) for i in range(cnt.value)]


def select_device(filter_text: str = ""):
    d = _DeviceDesc()
    _ck(lib().hetreco_select_device(filter_text.encode(), C.byref(d)))
    return DeviceDescriptor(d)


def select_from(candidates: Sequence[DeviceDescriptor], filter_text: str = "") -> int:
    arr = (_DeviceDesc * max(1, len(candidates)))()
    for i, c in enumerate(candidates):
        arr[i] = c._c()
    idx = C.c_int()
    _ck(lib().hetreco_select_from(arr, len(candidates), filter_text.encode(), C.byref(idx)))
    return idx.value


def describe_filter(filter_text: str) -> str:
    buf = C.create_string_buffer(512)
    _ck(lib().hetreco_filter_describe(filter_text.encode(), buf, 512))
    return buf.value.decode()


def cuda_device_count() -> int:
    n = C.c_int()
    _ck(lib().hetreco_cuda_device_count(C.byref(n)))
    return n.value


# ---------------------------------------------------------------------------
# pinned host memory
# ---------------------------------------------------------------------------


def pinned_empty(shape, dtype) -> np.ndarray:
    """Fortran-ordered numpy array in page-locked host memory (cudaHostAlloc)."""
    dtype = np.dtype(dtype)
    shape = tuple(int(s) for s in shape)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    p = C.c_void_p()
    _ck(lib().hetreco_host_alloc(nbytes, C.byref(p)))
    buf = (C.c_uint8 * max(nbytes, 1)).from_address(p.value)
    arr = np.frombuffer(buf, dtype=np.uint8, count=nbytes).view(dtype)
    arr = arr.reshape(shape, order="F")
    weakref.finalize(buf, lib().hetreco_host_free, C.c_void_p(p.value))
    return arr


# ---------------------------------------------------------------------------
# session (session.hpp)
# ---------------------------------------------------------------------------


class DataHandle:
    __slots__ = ("session_uid", "id")

    def __init__(self, session_uid=0, id=0):
        self.session_uid, self.id = int(session_uid), int(id)

    def valid(self):
        return self.id != 0

    def _c(self):
        return _Handle(self.session_uid, self.id)

    def __eq__(self, o):
        return isinstance(o, DataHandle) and (self.session_uid, self.id) == (o.session_uid, o.id)

    def __hash__(self):
        return hash((self.session_uid, self.id))

    def __repr__(self):
        return f"DataHandle({self.session_uid}, {self.id})"


class ComputeSession:
    """One selected device + device-resident data + kernels (session.hpp:48-137)."""

    def __init__(self, filter_text: str = "", device: DeviceDescriptor | None = None):
        self._h = C.c_void_p()
        if device is not None:
            _ck(lib().hetreco_session_create_on(device.backend_id.encode(), C.byref(self._h)))
        else:
            _ck(lib().hetreco_session_create(filter_text.encode(), C.byref(self._h)))

    def close(self):
        if self._h:
            _ck(lib().hetreco_session_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def device(self) -> DeviceDescriptor:
        d = _DeviceDesc()
        _ck(lib().hetreco_session_device(self._h, C.byref(d)))
        return DeviceDescriptor(d)

    # ---- data ----
    def register_data(self, data: Data | Sequence[np.ndarray], kind: DataKind | None = None) -> DataHandle:
        if not isinstance(data, Data):
            data = Data(data, kind if kind is not None else DataKind.Generic)
        arrs = [np.asfortranarray(a) for a in data.arrays]
        descs = _descs(arrs)
        h = _Handle()
        _ck(lib().hetreco_register_data(self._h, int(data.kind), len(arrs), descs, C.byref(h)))
        return DataHandle(h.session_uid, h.id)

    def allocate_data(self, shapes: Sequence[tuple], kind: DataKind = DataKind.Generic) -> DataHandle:
        """B200 extension: zero-filled device Data from (shape, dtype) pairs, no upload."""
        descs = (_ArrayDesc * max(1, len(shapes)))()
        for i, (shape, dt) in enumerate(shapes):
            descs[i] = _desc(shape, dt)
        h = _Handle()
        _ck(lib().hetreco_allocate_data(self._h, int(kind), len(shapes), descs, C.byref(h)))
        return DataHandle(h.session_uid, h.id)

    def layout_of(self, h: DataHandle) -> LayoutDescriptor:
        n, total, kind = C.c_int(), C.c_uint64(), C.c_int()
        _ck(lib().hetreco_session_layout(self._h, h._c(), None, 0, C.byref(n), C.byref(total), C.byref(kind)))
        out = (_ArrayDesc * max(1, n.value))()
        _ck(lib().hetreco_session_layout(self._h, h._c(), out, n.value, C.byref(n), C.byref(total), C.byref(kind)))
        return LayoutDescriptor([LayoutRecord(out[i]) for i in range(n.value)], total.value)

    def kind_of(self, h: DataHandle) -> DataKind:
        n, total, kind = C.c_int(), C.c_uint64(), C.c_int()
        _ck(lib().hetreco_session_layout(self._h, h._c(), None, 0, C.byref(n), C.byref(total), C.byref(kind)))
        return DataKind(kind.value)

    def fetch_data(self, h: DataHandle, out: Sequence[np.ndarray] | None = None) -> Data:
        layout = self.layout_of(h)
        if out is None:
            out = [np.empty(r.shape, dtype_of(r.element_type), order="F") for r in layout.records]
        ptrs = (C.c_void_p * max(1, len(out)))(*[a.ctypes.data for a in out])
        _ck(lib().hetreco_fetch_data(self._h, h._c(), len(out), ptrs))
        return Data(out, self.kind_of(h))

    def release_data(self, h: DataHandle):
        _ck(lib().hetreco_release_data(self._h, h._c()))

    def fetch_header_bytes(self, h: DataHandle) -> bytes:
        n = C.c_uint64()
        _ck(lib().hetreco_fetch_header_bytes(self._h, h._c(), None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        _ck(lib().hetreco_fetch_header_bytes(self._h, h._c(), buf, n.value, C.byref(n)))
        return bytes(buf)

    def copy_array(self, src: DataHandle, si: int, dst: DataHandle, di: int):
        _ck(lib().hetreco_copy_array(self._h, src._c(), si, dst._c(), di))

    def live_data_count(self) -> int:
        n = C.c_uint64()
        _ck(lib().hetreco_live_data_count(self._h, C.byref(n)))
        return n.value

    # ---- kernels ----
    def load_builtin_kernels(self):
        _ck(lib().hetreco_load_builtin_kernels(self._h))

    def kernel_names(self):
        buf = C.create_string_buffer(4096)
        _ck(lib().hetreco_kernel_names(self._h, buf, 4096))
        return [x for x in buf.value.decode().split("\n") if x]

    def load_kernels(self, units: Sequence[tuple[str, str]]):
        names = (C.c_char_p * max(1, len(units)))(*[u[0].encode() for u in units])
        srcs = (C.c_char_p * max(1, len(units)))(*[u[1].encode() for u in units])
        _ck(lib().hetreco_load_kernels(self._h, len(units), names, srcs))

    def launch_kernel(self, name: str, inp: DataHandle, out: DataHandle, params: bytes, global_size: int):
        pb = np.frombuffer(bytes(params) or b"\0", np.uint8)
        _ck(lib().hetreco_launch_kernel(self._h, name.encode(), inp._c(), out._c(), pb.ctypes.data, len(params),
                                        int(global_size)))

    def synchronize(self):
        _ck(lib().hetreco_synchronize(self._h))

    def timer_start(self):
        """Record a device timestamp on the session's compute stream."""
        _ck(lib().hetreco_session_timer_start(self._h))

    def timer_stop(self) -> float:
        """Seconds of device time since timer_start (waits for the stream)."""
        t = C.c_double()
        _ck(lib().hetreco_session_timer_stop(self._h, C.byref(t)))
        return t.value

    def counters(self):
        a, b = C.c_uint64(), C.c_uint64()
        _ck(lib().hetreco_counters(self._h, C.byref(a), C.byref(b)))
        return {"host_to_device": a.value, "device_to_host": b.value}

    def reset_counters(self):
        _ck(lib().hetreco_reset_counters(self._h))


# ---------------------------------------------------------------------------
# processes (process.hpp)
# ---------------------------------------------------------------------------


class ProcessParams:
    def __init__(self, values: dict | None = None):
        self._h = C.c_void_p()
        _ck(lib().hetreco_params_create(C.byref(self._h)))
        for k, v in (values or {}).items():
            self.set(k, v)

    def set(self, key: str, value):
        k = key.encode()
        if isinstance(value, bool):
            _ck(lib().hetreco_params_set_bool(self._h, k, int(value)))
        elif isinstance(value, (int, np.integer)):
            _ck(lib().hetreco_params_set_int(self._h, k, int(value)))
        elif isinstance(value, (float, np.floating)):
            _ck(lib().hetreco_params_set_real(self._h, k, float(value)))
        elif isinstance(value, str):
            _ck(lib().hetreco_params_set_string(self._h, k, value.encode()))
        else:
            raise TypeError(f"unsupported parameter type {type(value)}")
        return self

    def __del__(self):
        try:
            if self._h:
                lib().hetreco_params_destroy(self._h)
        except Exception:
            pass


class LaunchStats:
    def __init__(self, init_calls, launches, last, total, init_s):
        self.init_calls, self.launches = init_calls, launches
        self.last_launch_seconds, self.total_launch_seconds, self.init_seconds = last, total, init_s

    def mean_launch_seconds(self):
        return 0.0 if self.launches == 0 else self.total_launch_seconds / self.launches


class Process:
    """A builtin process ("negate", "fft2d", "complex_element_prod",
    "ximage_sum", "rss_combine", "sens_recon", "rss_recon")."""

    def __init__(self, session: ComputeSession, kind: str, name: str | None = None, _handle=None):
        self.session = session
        self.kind = kind
        self._owner = True
        if _handle is not None:
            self._h = _handle
            self._owner = False
        else:
            self._h = C.c_void_p()
            _ck(lib().hetreco_process_create(session._h, kind.encode(), (name or kind).encode(),
                                             C.byref(self._h)))

    def __del__(self):
        try:
            if self._owner and self._h:
                lib().hetreco_process_destroy(self._h)
        except Exception:
            pass

    def set_input(self, h: DataHandle):
        _ck(lib().hetreco_process_set_input(self._h, h._c()))
        return self

    def set_output(self, h: DataHandle):
        _ck(lib().hetreco_process_set_output(self._h, h._c()))
        return self

    def init(self, params: dict | ProcessParams | None = None):
        if isinstance(params, dict):
            params = ProcessParams(params)
        _ck(lib().hetreco_process_init(self._h, params._h if params is not None else None))
        return self

    def launch(self):
        _ck(lib().hetreco_process_launch(self._h))

    def state(self) -> str:
        s = C.c_int()
        _ck(lib().hetreco_process_state(self._h, C.byref(s)))
        return "initialized" if s.value else "created"

    def profile(self, reps: int = 5):
        """Mean device seconds of each kernel of this process (record order)."""
        n = C.c_int()
        buf = (C.c_double * 4096)()
        _ck(lib().hetreco_process_profile(self._h, reps, buf, 4096, C.byref(n)))
        return [buf[i] for i in range(n.value)]

    def stats(self) -> LaunchStats:
        a, b = C.c_uint64(), C.c_uint64()
        c, d, e = C.c_double(), C.c_double(), C.c_double()
        _ck(lib().hetreco_process_stats(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d), C.byref(e)))
        return LaunchStats(a.value, b.value, c.value, d.value, e.value)


def chain(session: ComputeSession, name: str, stages: Sequence[Process]) -> Process:
    """CompositeProcess over `stages` (process.hpp:122-140); the chain takes
    ownership of the stages (their Python objects remain usable as views)."""
    arr = (C.c_void_p * max(1, len(stages)))(*[s._h for s in stages])
    h = C.c_void_p()
    _ck(lib().hetreco_chain_create(session._h, name.encode(), arr, len(stages), C.byref(h)))
    for s in stages:
        s._owner = False
    comp = Process(session, "chain", _handle=h)
    comp._owner = True
    comp._stages = list(stages)
    return comp


# ---------------------------------------------------------------------------
# pinned streaming (paper §III-A2)
# ---------------------------------------------------------------------------


class StreamingRecon:
    def __init__(self, session: ComputeSession, method: str, nx: int, ny: int, coils: int, chunk_frames: int,
                 smaps: np.ndarray | None = None, shift: bool = False):
        self.session = session
        self.method = method
        self._smaps = None if smaps is None else np.asfortranarray(smaps, dtype=np.complex64)
        self._h = C.c_void_p()
        m = 0 if method == "sense" else 1
        _ck(lib().hetreco_stream_create(session._h, m, nx, ny, coils, chunk_frames,
                                        self._smaps.ctypes.data if self._smaps is not None else None, int(shift),
                                        C.byref(self._h)))
        self.nx, self.ny, self.coils = nx, ny, coils

    def run(self, kspace: np.ndarray, out: np.ndarray):
        assert kspace.flags.f_contiguous and out.flags.f_contiguous
        frames = kspace.size // (self.nx * self.ny * self.coils)
        _ck(lib().hetreco_stream_run(self._h, kspace.ctypes.data, frames, out.ctypes.data))
        return out

    def __del__(self):
        try:
            if self._h:
                lib().hetreco_stream_destroy(self._h)
        except Exception:
            pass


def frame_slab(index: int, count: int, frames: int) -> tuple[int, int]:
    """[begin, end) frames of slab `index` of `count` (the library's partition)."""
    b, e = C.c_uint64(), C.c_uint64()
    _ck(lib().hetreco_frame_slab(index, count, frames, C.byref(b), C.byref(e)))
    return b.value, e.value


class MultiGpuRecon:
    """One host k-space volume reconstructed over several GPUs by frame slab
    (hetreco_multi_*): one worker thread, session and streaming pipeline per
    backend id, each moving its own contiguous slab; no collective."""

    def __init__(self, backend_ids: Sequence[str], method: str, nx: int, ny: int, coils: int, chunk_frames: int,
                 smaps: np.ndarray | None = None, shift: bool = False, bind_numa: bool = True):
        self.method = method
        self.nx, self.ny, self.coils = nx, ny, coils
        self.backend_ids = list(backend_ids)
        smp = None if smaps is None else np.asfortranarray(smaps, dtype=np.complex64)
        ids = (C.c_char_p * max(1, len(self.backend_ids)))(*[b.encode() for b in self.backend_ids])
        self._h = C.c_void_p()
        m = 0 if method == "sense" else 1
        _ck(lib().hetreco_multi_create(len(self.backend_ids), ids, m, nx, ny, coils, chunk_frames,
                                       smp.ctypes.data if smp is not None else None, int(shift), int(bind_numa),
                                       C.byref(self._h)))

    def run(self, kspace: np.ndarray, out: np.ndarray):
        assert kspace.flags.f_contiguous and out.flags.f_contiguous
        frames = kspace.size // (self.nx * self.ny * self.coils)
        _ck(lib().hetreco_multi_run(self._h, kspace.ctypes.data, frames, out.ctypes.data))
        return out

    def slabs(self) -> list[dict]:
        """Per slab of the last run: backend id, first frame, frames, seconds."""
        res = []
        for i, bid in enumerate(self.backend_ids):
            f, n, t = C.c_uint64(), C.c_uint64(), C.c_double()
            _ck(lib().hetreco_multi_slab(self._h, i, C.byref(f), C.byref(n), C.byref(t)))
            res.append({"backend_id": bid, "first_frame": f.value, "frames": n.value, "seconds": t.value})
        return res

    def close(self):
        if self._h:
            _ck(lib().hetreco_multi_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# layer 1: the Backend contract on one GPU (backend.hpp:44-79)
# ---------------------------------------------------------------------------


class CudaBackend:
    def __init__(self, ordinal: int = 0, capacity_bytes: int = 0):
        self._h = C.c_void_p()
        _ck(lib().hetreco_cuda_backend_create(ordinal, capacity_bytes, C.byref(self._h)))

    def close(self):
        if self._h:
            _ck(lib().hetreco_cuda_backend_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def device(self) -> DeviceDescriptor:
        d = _DeviceDesc()
        _ck(lib().hetreco_cuda_backend_device(self._h, C.byref(d)))
        return DeviceDescriptor(d)

    def allocate(self, nbytes: int) -> int:
        b = C.c_uint64()
        _ck(lib().hetreco_cuda_allocate(self._h, nbytes, C.byref(b)))
        return b.value

    def release(self, buf: int):
        _ck(lib().hetreco_cuda_release(self._h, buf))

    def upload(self, buf: int, offset: int, data: bytes | np.ndarray):
        a = np.frombuffer(bytes(data), np.uint8) if not isinstance(data, np.ndarray) else data
        _ck(lib().hetreco_cuda_upload(self._h, buf, offset, a.ctypes.data, a.nbytes))

    def download(self, buf: int, offset: int, nbytes: int) -> bytes:
        a = np.empty(nbytes, np.uint8)
        _ck(lib().hetreco_cuda_download(self._h, buf, offset, a.ctypes.data, nbytes))
        return a.tobytes()

    def copy(self, src, so, dst, do, n):
        _ck(lib().hetreco_cuda_copy(self._h, src, so, dst, do, n))

    @staticmethod
    def intrinsic_kernel_names():
        n = C.c_int()
        _ck(lib().hetreco_cuda_kernel_count(C.byref(n)))
        return [lib().hetreco_cuda_kernel_name(i).decode() for i in range(n.value)]

    def execute(self, name, inp, inp_hdr, out, out_hdr, params: bytes, global_size: int):
        pb = np.frombuffer(bytes(params) or b"\0", np.uint8)
        _ck(lib().hetreco_cuda_execute(self._h, name.encode(), inp, inp_hdr, out, out_hdr, pb.ctypes.data,
                                       len(params), global_size))

    def synchronize(self):
        _ck(lib().hetreco_cuda_synchronize(self._h))


def version() -> str:
    return lib().hetreco_version().decode()


# ---------------------------------------------------------------------------
# io: MAT v5 / PGM-PPM / raw+sidecar (SPEC.md io module; include/hetreco_b200/io.hpp)
# ---------------------------------------------------------------------------


def _take_vars(m) -> list:
    """Copies the variables of a native list into Fortran-ordered numpy arrays."""
    L = lib()
    try:
        n = C.c_int()
        _ck(L.hetreco_mat_count(m, C.byref(n)))
        out = []
        for i in range(n.value):
            d = _ArrayDesc()
            name = C.create_string_buffer(256)
            _ck(L.hetreco_mat_variable(m, i, name, 256, C.byref(d)))
            shape = tuple(int(d.dims[k]) for k in range(d.rank))
            dt = np.dtype(dtype_of(d.element_type))
            nbytes = int(np.prod(shape)) * dt.itemsize
            buf = (C.c_char * nbytes).from_address(d.host)
            a = np.frombuffer(buf, dtype=dt).reshape(shape, order="F").copy(order="F")
            out.append((name.value.decode(errors="replace"), a))
        return out
    finally:
        L.hetreco_mat_free(m)


def read_mat(path: str) -> dict:
    """read_mat: {name: array} in file order."""
    m = C.c_void_p()
    _ck(lib().hetreco_mat_read(os.fsencode(path), 0, C.byref(m)))
    return dict(_take_vars(m))


def parse_mat(data: bytes) -> dict:
    m = C.c_void_p()
    buf = C.create_string_buffer(bytes(data), len(data))
    _ck(lib().hetreco_mat_parse(buf, len(data), 0, C.byref(m)))
    return dict(_take_vars(m))


def write_mat(path: str, variables) -> None:
    """write_mat; variables = {name: array} or [(name, array)]."""
    items = list(variables.items()) if isinstance(variables, dict) else list(variables)
    arrays = [np.asfortranarray(a) for _, a in items]
    names = (C.c_char_p * max(1, len(items)))(*[str(n).encode() for n, _ in items])
    _ck(lib().hetreco_mat_write(os.fsencode(path), len(items), names, _descs(arrays)))


def read_image(path: str) -> np.ndarray:
    """PGM (P5) -> uint8 [w, h]; PPM (P6) -> uint8 [3, w, h]."""
    m = C.c_void_p()
    _ck(lib().hetreco_image_read(os.fsencode(path), 0, C.byref(m)))
    return _take_vars(m)[0][1]


def write_image(path: str, image: np.ndarray) -> None:
    a = np.asfortranarray(image)
    _ck(lib().hetreco_image_write(os.fsencode(path), C.byref(_desc(a.shape, a.dtype, a.ctypes.data))))


def read_raw(path: str, sidecar_path: str) -> np.ndarray:
    m = C.c_void_p()
    _ck(lib().hetreco_raw_read(os.fsencode(path), os.fsencode(sidecar_path), 0, C.byref(m)))
    return _take_vars(m)[0][1]


def write_raw(path: str, sidecar_path: str, array: np.ndarray) -> None:
    a = np.asfortranarray(array)
    _ck(lib().hetreco_raw_write(os.fsencode(path), os.fsencode(sidecar_path),
                                C.byref(_desc(a.shape, a.dtype, a.ctypes.data))))


def gen_phantom(session: "ComputeSession", nx: int = 128, ny: int = 128, frames: int = 16, coils: int = 8,
                seed: int = 1):
    """gen_phantom on the session's device -> (kdata Y, smaps S, truth M)."""
    Y = np.empty((nx, ny, coils, frames), np.complex64, order="F")
    S = np.empty((nx, ny, coils), np.complex64, order="F")
    M = np.empty((nx, ny, frames), np.complex64, order="F")
    _ck(lib().hetreco_gen_phantom(session._h, nx, ny, frames, coils, seed, Y.ctypes.data, S.ctypes.data,
                                  M.ctypes.data))
    return Y, S, M


def phantom_blobs(nx: int, ny: int, seed: int):
    """The seeded blob parameters gen_phantom uses: [(amp, radius, angle, sigma)] x 3."""
    out = (C.c_double * 12)()
    _ck(lib().hetreco_phantom_blobs(nx, ny, seed, out))
    return [tuple(out[4 * i: 4 * i + 4]) for i in range(3)]


# ---------------------------------------------------------------------------
# source kernels (NVRTC, sm_100a)
# ---------------------------------------------------------------------------


def nvrtc_available() -> bool:
    v = C.c_int()
    _ck(lib().hetreco_nvrtc_available(C.byref(v)))
    return bool(v.value)


def compile_check(unit_name: str, source: str):
    """Compile one kernel-source unit for sm_100a without a device; returns
    (kernel names, compiler log).  Raises CompileError with the log."""
    names = C.create_string_buffer(4096)
    log = C.create_string_buffer(65536)
    rc = lib().hetreco_nvrtc_compile_check(unit_name.encode(), source.encode(), names, 4096, log, 65536)
    if rc != 0:
        msg = lib().hetreco_last_error().decode(errors="replace")
        raise ERRORS.get(rc, HetrecoError)(msg)
    return [n for n in names.value.decode().split("\n") if n], log.value.decode(errors="replace")


# ---------------------------------------------------------------------------
# NUMA placement (multi-GPU streaming, SURVEY.md §8 e)
# ---------------------------------------------------------------------------


def device_numa_node(ordinal: int) -> int:
    n = C.c_int()
    _ck(lib().hetreco_device_numa_node(ordinal, C.byref(n)))
    return n.value


def bind_numa_node(node: int) -> int:
    """Restricts the calling thread (and later threads) to the CPUs of `node`."""
    n = C.c_int()
    _ck(lib().hetreco_bind_numa_node(node, C.byref(n)))
    return n.value


def bind_to_device_numa(ordinal: int) -> int:
    """Binds the calling thread to its GPU's NUMA node; returns the node (-1: none)."""
    node = device_numa_node(ordinal)
    bind_numa_node(node)
    return node


def parse_cpulist(text: str) -> list:
    buf = (C.c_int * 4096)()
    n = C.c_int()
    _ck(lib().hetreco_parse_cpulist(text.encode(), buf, 4096, C.byref(n)))
    return list(buf[: min(n.value, 4096)])
