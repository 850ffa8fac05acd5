/*
 * hetreco_b200.h -- C-ABI of the B200 build (libhetreco_b200.so).
 *
 * Plain C types only (pointers, sizes, fixed-width integers); every function
 * returns a status (0 = ok, else the hetreco::ErrorCode value of the
 * exception the C++ layer raised) and the message is available from
 * hetreco_last_error() on the calling thread.  Each entry point names the
 * reference interface it replaces (paths relative to
 * /root/reference/proj/core).  INTEGRATION.md shows the reference-side
 * bindings (a C++ Backend adapter, and the ctypes stub the tests use).
 *
 * Two layers:
 *   1. hetreco_cuda_*  -- the Backend contract (include/hetreco/backend.hpp:44-79)
 *      on one GPU: buffers, transfers, builtin kernel execution.  A reference
 *      build gains the B200 by registering an adapter over these.
 *   2. hetreco_session_* / hetreco_process_* / hetreco_stream_* -- the
 *      operator API (session.hpp, process.hpp) implemented natively, with
 *      the fused sm_100a reconstruction processes and the pinned streaming
 *      pipeline.
 */
#ifndef HETRECO_B200_H
#define HETRECO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The library is built with -fvisibility=hidden: only this C-ABI is exported
 * (its C++ internals share the hetreco:: namespace with the reference and
 * must not interpose on a reference build loaded in the same process). */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* ---- errors (include/hetreco/errors.hpp:12-219) ----------------------------- */
#define HETRECO_OK 0
const char* hetreco_last_error(void);
/* Version string of this build. */
const char* hetreco_version(void);

/* ---- devices (include/hetreco/device.hpp:37-114; src/device.cpp:106-218) ----- */
typedef struct hetreco_device_desc {
    char backend_id[32];
    uint32_t device_index;
    int32_t device_type; /* 0 cpu, 1 gpu, 2 accelerator (DeviceType order) */
    char vendor[32];
    char name[128];
    char api_version[16];
    uint64_t global_memory_bytes;
    uint64_t base_alignment_bytes;
    int32_t supports_source_kernels;
} hetreco_device_desc;

/* enumerate_devices (device.hpp:94); writes up to `cap` entries, *count = total */
int hetreco_enumerate_devices(hetreco_device_desc* out, int cap, int* count);
/* select_device(DeviceFilter::parse(filter_text)) (device.hpp:103, :76-80) */
int hetreco_select_device(const char* filter_text, hetreco_device_desc* out);
/* select_from on a caller-supplied candidate list (device.hpp:111-114); *index = winner */
int hetreco_select_from(const hetreco_device_desc* candidates, int n, const char* filter_text, int* index);

/* ---- layer 1: the Backend contract on one GPU (backend.hpp:44-79) ------------ */
typedef struct hetreco_cuda_backend_t* hetreco_cuda_backend;

/* Number of visible CUDA devices (replaces the backend list, backend.cpp:294-313). */
int hetreco_cuda_device_count(int* count);
/* A standalone backend on GPU `ordinal`; capacity_bytes 0 = unlimited
 * (make_reference_backend(capacity), backend.hpp:91-96). */
int hetreco_cuda_backend_create(int ordinal, uint64_t capacity_bytes, hetreco_cuda_backend* out);
int hetreco_cuda_backend_destroy(hetreco_cuda_backend b);
/* Backend::devices() (backend.hpp:48) */
int hetreco_cuda_backend_device(hetreco_cuda_backend b, hetreco_device_desc* out);
/* Backend::allocate / release (backend.hpp:52-53); zero-filled */
int hetreco_cuda_allocate(hetreco_cuda_backend b, uint64_t bytes, uint64_t* buffer_id);
int hetreco_cuda_release(hetreco_cuda_backend b, uint64_t buffer_id);
/* Backend::upload / download (backend.hpp:54-57); synchronous on the host span */
int hetreco_cuda_upload(hetreco_cuda_backend b, uint64_t buffer_id, uint64_t offset, const void* src, uint64_t bytes);
int hetreco_cuda_download(hetreco_cuda_backend b, uint64_t buffer_id, uint64_t offset, void* dst, uint64_t bytes);
/* Backend::copy (backend.hpp:59-60) */
int hetreco_cuda_copy(hetreco_cuda_backend b, uint64_t src, uint64_t src_offset, uint64_t dst, uint64_t dst_offset,
                      uint64_t bytes);
/* Backend::intrinsic_kernels (backend.hpp:63): names of the builtin kernels */
int hetreco_cuda_kernel_count(int* count);
const char* hetreco_cuda_kernel_name(int index);
/* Backend::execute (backend.hpp:74-75) with KernelBinding (backend.hpp:26-32):
 * buffers by id; `params` is copied before return (the reference borrows it). */
int hetreco_cuda_execute(hetreco_cuda_backend b, const char* kernel_name, uint64_t input, uint64_t input_header,
                         uint64_t output, uint64_t output_header, const void* params, uint64_t params_size,
                         uint64_t global_size);
/* Backend::synchronize (backend.hpp:78); surfaces device faults */
int hetreco_cuda_synchronize(hetreco_cuda_backend b);
/* supports_source_kernels (backend.hpp:51): 1 when NVRTC is available */
int hetreco_cuda_supports_source(hetreco_cuda_backend b, int* yes);
/* compile (backend.hpp:71): kernel-source units -> NVRTC sm_100a cubins,
 * loaded into this backend.  out = one "unit_tag\tkernel_name\n" line per
 * kernel (unit_tag identifies the compiled unit for execute_unit).
 * CompileError carries the units' compiler logs. */
int hetreco_cuda_compile(hetreco_cuda_backend b, int count, const char* const* unit_names, const char* const* sources,
                         char* out, uint64_t cap);
/* execute (backend.hpp:74-75) of a kernel returned by hetreco_cuda_compile */
int hetreco_cuda_execute_unit(hetreco_cuda_backend b, const char* unit_tag, const char* kernel_name, uint64_t input,
                              uint64_t input_header, uint64_t output, uint64_t output_header, const void* params,
                              uint64_t params_size, uint64_t global_size);
/* Page-locked host memory for full-rate DMA (the paper's pinned buffers). */
int hetreco_host_alloc(uint64_t bytes, void** out);
int hetreco_host_free(void* p);

/* ---- layer 2: sessions (session.hpp:18-137; src/session.cpp) ------------------ */
typedef struct hetreco_session_t* hetreco_session;
typedef struct hetreco_handle {
    uint64_t session_uid;
    uint64_t id;
} hetreco_handle; /* DataHandle, session.hpp:18-24 */

/* One array of a Data set (NDArray, ndarray.hpp:70-122; LayoutRecord, layout.hpp:17-28). */
typedef struct hetreco_array_desc {
    uint64_t element_type; /* ElementType code 1..6 */
    uint32_t rank;
    uint32_t _pad;
    uint64_t dims[8];
    uint64_t offset_bytes; /* filled by hetreco_session_layout */
    void* host;            /* host payload (register) / destination (fetch) */
} hetreco_array_desc;

/* DataKind (ndarray.hpp:125-129) */
#define HETRECO_XDATA 0
#define HETRECO_KDATA 1
#define HETRECO_GENERIC 2

/* ComputeSession(DeviceFilter::parse(text)) -- one-call setup (session.hpp:55) */
int hetreco_session_create(const char* filter_text, hetreco_session* out);
/* ComputeSession(DeviceDescriptor) for a backend id such as "cuda3" (session.hpp:58) */
int hetreco_session_create_on(const char* backend_id, hetreco_session* out);
int hetreco_session_destroy(hetreco_session s);
int hetreco_session_device(hetreco_session s, hetreco_device_desc* out);
/* register_data (session.hpp:73; session.cpp:60-83): arrays[i].host = payload */
int hetreco_register_data(hetreco_session s, int kind, int count, const hetreco_array_desc* arrays,
                          hetreco_handle* out);
/* B200 extension: allocate a zero-filled device Data set without uploading. */
int hetreco_allocate_data(hetreco_session s, int kind, int count, const hetreco_array_desc* arrays,
                          hetreco_handle* out);
/* layout_of (session.hpp:77): *count arrays; fills up to cap records and *total_bytes */
int hetreco_session_layout(hetreco_session s, hetreco_handle h, hetreco_array_desc* out, int cap, int* count,
                           uint64_t* total_bytes, int* kind);
/* fetch_data (session.hpp:74; session.cpp:85-98) into caller buffers dst[i] */
int hetreco_fetch_data(hetreco_session s, hetreco_handle h, int count, void* const* dst);
/* release_data (session.hpp:75) */
int hetreco_release_data(hetreco_session s, hetreco_handle h);
/* fetch_header_bytes (session.hpp:82-84); *n = header length */
int hetreco_fetch_header_bytes(hetreco_session s, hetreco_handle h, void* dst, uint64_t cap, uint64_t* n);
/* copy_array (session.hpp:86-89) */
int hetreco_copy_array(hetreco_session s, hetreco_handle src, uint64_t src_index, hetreco_handle dst,
                       uint64_t dst_index);
/* load_builtin_kernels / kernels().names() (session.hpp:94-101); names '\n'-joined */
int hetreco_load_builtin_kernels(hetreco_session s);
int hetreco_kernel_names(hetreco_session s, char* buf, uint64_t cap);
/* load_kernels(units) (session.hpp:97): kernel-source units (the reference's
 * HETRECO_KERNEL dialect) compiled by NVRTC for sm_100a; CompileError carries
 * every failing unit's log, DuplicateKernel leaves the registry unchanged. */
int hetreco_load_kernels(hetreco_session s, int count, const char* const* unit_names, const char* const* sources);
/* launch_kernel (session.hpp:108-109; session.cpp:154-169) */
int hetreco_launch_kernel(hetreco_session s, const char* name, hetreco_handle in, hetreco_handle out,
                          const void* params, uint64_t params_size, uint64_t global_size);
int hetreco_synchronize(hetreco_session s);
/* counters / reset_counters (session.hpp:115-116) */
int hetreco_counters(hetreco_session s, uint64_t* host_to_device, uint64_t* device_to_host);
int hetreco_reset_counters(hetreco_session s);
int hetreco_live_data_count(hetreco_session s, uint64_t* n);

/* ---- layer 2: processes (process.hpp:21-140) ---------------------------------- */
typedef struct hetreco_params_t* hetreco_params;
typedef struct hetreco_process_t* hetreco_process;

/* ProcessParams (process.hpp:21-52) */
int hetreco_params_create(hetreco_params* out);
int hetreco_params_destroy(hetreco_params p);
int hetreco_params_set_bool(hetreco_params p, const char* key, int value);
int hetreco_params_set_int(hetreco_params p, const char* key, int64_t value);
int hetreco_params_set_real(hetreco_params p, const char* key, double value);
int hetreco_params_set_string(hetreco_params p, const char* key, const char* value);

/* Builtin process by kind: "negate", "fft2d", "complex_element_prod",
 * "ximage_sum", "rss_combine", "sens_recon", "rss_recon". */
int hetreco_process_create(hetreco_session s, const char* kind, const char* name, hetreco_process* out);
/* chain(stages) (process.hpp:138-140); takes ownership of the stage handles
 * (they must not be destroyed separately afterwards). */
int hetreco_chain_create(hetreco_session s, const char* name, hetreco_process* stages, int n, hetreco_process* out);
int hetreco_process_destroy(hetreco_process p);
int hetreco_process_set_input(hetreco_process p, hetreco_handle h);
int hetreco_process_set_output(hetreco_process p, hetreco_handle h);
/* init (process.hpp:94): plans baked, device work captured in a CUDA graph */
int hetreco_process_init(hetreco_process p, hetreco_params params /* may be NULL */);
/* launch (process.hpp:95): one cudaGraphLaunch, asynchronous */
int hetreco_process_launch(hetreco_process p);
/* state (0 created, 1 initialized) and LaunchStats (process.hpp:55-64) */
int hetreco_process_state(hetreco_process p, int* state);
int hetreco_process_stats(hetreco_process p, uint64_t* init_calls, uint64_t* launches, double* last_launch_s,
                          double* total_launch_s, double* init_s);
/* Per-kernel device time: launches the recorded work `reps` times without the
 * graph, CUDA events between kernels on the compute stream; writes the mean
 * seconds of each kernel (record order) and *n = kernel count. */
int hetreco_process_profile(hetreco_process p, int reps, double* kernel_seconds, int cap, int* n);
/* Device timer on the session's compute stream (events bracket the region). */
int hetreco_session_timer_start(hetreco_session s);
int hetreco_session_timer_stop(hetreco_session s, double* seconds);
/* CompositeProcess::stage (process.hpp:128): borrowed pointer */
int hetreco_chain_stage(hetreco_process chain, int index, hetreco_process* out);

/* ---- layer 2: pinned host streaming (paper §III-A2 pinned/mapped transfers) ---- */
typedef struct hetreco_stream_t* hetreco_stream;
#define HETRECO_METHOD_SENSE 0
#define HETRECO_METHOD_RSS 1
int hetreco_stream_create(hetreco_session s, int method, uint64_t nx, uint64_t ny, uint64_t coils,
                          uint64_t chunk_frames, const void* host_smaps, int shift, hetreco_stream* out);
/* host_kspace [nx,ny,coils,frames] c64 -> host_out [nx,ny,frames]; blocks */
int hetreco_stream_run(hetreco_stream st, const void* host_kspace, uint64_t frames, void* host_out);
int hetreco_stream_destroy(hetreco_stream st);

/* ---- layer 2: one host volume over several GPUs by frame slab (SURVEY §8 e) ----
 * No reference counterpart: the reference binds one device per session and has
 * no multi-device path.  Slab g of G = frames
 * [floor(g F / G), floor((g+1) F / G)); one worker thread + ComputeSession +
 * streaming pipeline per entry of backend_ids (ids may repeat); no collective. */
typedef struct hetreco_multi_t* hetreco_multi;
int hetreco_frame_slab(uint64_t index, uint64_t count, uint64_t frames, uint64_t* begin, uint64_t* end);
int hetreco_multi_create(int n, const char* const* backend_ids, int method, uint64_t nx, uint64_t ny, uint64_t coils,
                         uint64_t chunk_frames, const void* host_smaps, int shift, int bind_numa, hetreco_multi* out);
/* host_kspace [nx,ny,coils,frames] c64 -> host_out [nx,ny,frames]; blocks */
int hetreco_multi_run(hetreco_multi m, const void* host_kspace, uint64_t frames, void* host_out);
/* slab `index` of the last run: first frame, frame count, host seconds */
int hetreco_multi_slab(hetreco_multi m, int index, uint64_t* first, uint64_t* frames, double* seconds);
int hetreco_multi_device_count(hetreco_multi m, int* n);
int hetreco_multi_destroy(hetreco_multi m);

/* ---- host-only helpers (layout.hpp:37-65): pack + header wire format ----------- */
/* pack(Data, alignment) then serialize_layout_header: writes (1+11*count) u64
 * words to `words` (cap in words) and offsets into arrays[i].offset_bytes. */
int hetreco_pack_layout(int count, hetreco_array_desc* arrays, uint64_t alignment, uint64_t* words, uint64_t cap,
                        uint64_t* total_bytes);
/* parse_layout_header: fills up to cap arrays; *count, *alignment, *total_bytes */
int hetreco_parse_layout_header(const void* bytes, uint64_t nbytes, hetreco_array_desc* out, int cap, int* count,
                                uint64_t* alignment, uint64_t* total_bytes);
/* DeviceFilter::parse + describe (device.hpp:76-86) */
int hetreco_filter_describe(const char* filter_text, char* buf, uint64_t cap);

/* ---- io: MAT v5 / PGM-PPM / raw+sidecar (SPEC.md io module :470-533) ----
 * Readers return a variable list; payloads stay owned by it (and are
 * page-locked when pinned != 0, ready for register_data / hetreco_stream_run
 * DMA) until hetreco_mat_free.  Error codes 22..26: MalformedFile,
 * UnsupportedFeature (message names the feature), IoError, SizeMismatch,
 * MalformedSidecar. */
typedef struct hetreco_mat_t* hetreco_mat;
/* read_mat(path) */
int hetreco_mat_read(const char* path, int pinned, hetreco_mat* out);
/* the same parser over an in-memory file image */
int hetreco_mat_parse(const void* bytes, uint64_t size, int pinned, hetreco_mat* out);
/* read_image: one variable "image", UINT8 [w,h] (P5) or [3,w,h] (P6) */
int hetreco_image_read(const char* path, int pinned, hetreco_mat* out);
/* read_raw: one variable "raw" */
int hetreco_raw_read(const char* path, const char* sidecar_path, int pinned, hetreco_mat* out);
int hetreco_mat_count(hetreco_mat m, int* count);
/* variable `index`: name (NUL-terminated into name[cap]) and desc (type, rank,
 * dims, host = payload pointer, offset_bytes = 1 when page-locked) */
int hetreco_mat_variable(hetreco_mat m, int index, char* name, uint64_t cap, hetreco_array_desc* desc);
int hetreco_mat_free(hetreco_mat m);
/* write_mat(path, variables); arrays[i].host = payload */
int hetreco_mat_write(const char* path, int count, const char* const* names, const hetreco_array_desc* arrays);
/* write_image (UINT8, or FLOAT32 in [0,1] -> round(v*255)) */
int hetreco_image_write(const char* path, const hetreco_array_desc* image);
int hetreco_raw_write(const char* path, const char* sidecar_path, const hetreco_array_desc* array);

/* ---- gen_phantom ----------------------------
 * Seeded synthetic cine on the session's device: truth = 3 rotating Gaussian
 * blobs, smaps = normalised complex coil maps (sum |S|^2 = 1), kdata =
 * F(S . truth).  Host outputs (COMPLEX64, column-major) may be NULL:
 * kdata [nx,ny,coils,frames], smaps [nx,ny,coils], truth [nx,ny,frames].
 * InvalidParams unless nx, ny are powers of two in [2, 4096]. */
int hetreco_gen_phantom(hetreco_session s, uint64_t nx, uint64_t ny, uint64_t frames, uint64_t coils,
                        uint64_t seed, void* kdata, void* smaps, void* truth);
/* the seeded blob parameters (amp, radius, angle, sigma) x 3 -- host only */
int hetreco_phantom_blobs(uint64_t nx, uint64_t ny, uint64_t seed, double* out12);

/* ---- source kernels (cpujit_backend.cpp:121-177 role) --------
 * Compile one unit with NVRTC for sm_100a without loading it (no device
 * needed): names = its kernels, '\n'-joined; log = compiler output (the
 * failure log on CompileError). */
int hetreco_nvrtc_compile_check(const char* unit_name, const char* source, char* names, uint64_t names_cap,
                                char* log, uint64_t log_cap);
int hetreco_nvrtc_available(int* available);

/* ---- NUMA placement for multi-GPU streaming (SURVEY.md §8 e) ------------------
 * Each rank binds its host thread to the NUMA node of its GPU before
 * allocating the pinned slab it streams from (first-touch placement). */
int hetreco_device_numa_node(int ordinal, int* node);       /* -1: no NUMA info */
int hetreco_bind_numa_node(int node, int* cpus);            /* node < 0: no-op */
int hetreco_parse_cpulist(const char* text, int* cpus, int cap, int* count);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif
