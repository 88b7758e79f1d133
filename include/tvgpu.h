/*
 * tvgpu.h — C ABI of libtvgpu.so, the B200 data path behind the treevault-compatible
 * checkpointing API in paper_2605_23066_b200/.
 *
 * The reference (treevault, /root/reference/pkg/src/treevault) is pure Python + numpy and
 * has no FFI of its own.  Each entry point below replaces one Python seam of the
 * reference's hot path; the seam it replaces is cited beside it (file:line relative to
 * /root/reference/pkg/src/treevault).  INTEGRATION.md shows the ctypes binding a
 * maintainer of the reference would add, and paper_2605_23066_b200/native.py is the
 * binding this package uses.
 *
 * Conventions
 *   - Every function returns an int status: TV_OK (0) or a negative TV_ERR_* code.
 *     tv_last_error() copies the message of the calling thread's last failure.
 *   - All buffers are caller-owned.  Device addresses are plain uint64 CUDA UVA
 *     addresses (torch tensors' data_ptr(), peer-mapped or IPC-opened pointers);
 *     streams are cudaStream_t passed as void*.
 *   - Arrays are row-major and contiguous; a box is (origin, extent) per dimension,
 *     exactly the reference's `ranges` tuples (sharding.py:21, Range = (offset, extent)).
 *   - No torch types cross this boundary.
 */
#ifndef TVGPU_H
#define TVGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TV_ABI_VERSION 2
#define TV_MAX_RANK 8

#define TV_OK 0
#define TV_ERR_CUDA (-1)   /* CUDA runtime / kernel launch failure               */
#define TV_ERR_IO (-2)     /* open/pwrite/pread/rename failure                   */
#define TV_ERR_ARG (-3)    /* malformed descriptor                               */
#define TV_ERR_NOMEM (-4)  /* pinned / device staging allocation failed          */
#define TV_ERR_STATE (-5)  /* engine misuse (e.g. wrong device)                  */

/* Element types of converting copies (tv_copy.src_dtype / dst_dtype). */
#define TV_DT_RAW 0        /* no conversion: bytes are copied                     */
#define TV_DT_F32 1
#define TV_DT_F64 2
#define TV_DT_I32 3
#define TV_DT_I64 4
#define TV_DT_U8 5
#define TV_DT_BOOL 6
#define TV_DT_BF16 7

/* Bits a converting copy ORs into its flags word (treemodel.py:417-441 checks). */
#define TV_CAST_OVERFLOW 1u     /* integer narrowing / float->int out of range         */
#define TV_CAST_NONINTEGRAL 2u  /* float->int of a non-integral value                  */
#define TV_CAST_NONFINITE 4u    /* float->int of inf / nan                              */

/* A box inside one row-major array. */
typedef struct tv_array_box {
  uint64_t base;                /* address of element (0,…,0) of the array           */
  int64_t shape[TV_MAX_RANK];   /* array extents                                      */
  int64_t off[TV_MAX_RANK];     /* box origin inside the array                        */
} tv_array_box;

/* One N-d box copy src → dst (same extents).  Pack is dst = a dense box of shape ext,
 * unpack is src = a dense box; both sides may be strided (reshard scatter).
 * With src_dtype != TV_DT_RAW the copy converts element types on the fly (the load-time
 * cast of treemodel.py:444-484 fused into the unpack): round-to-nearest-even float
 * narrowing, checked integer narrowing; violations are OR-ed into *flags. */
typedef struct tv_copy {
  tv_array_box src;
  tv_array_box dst;
  int64_t ext[TV_MAX_RANK];
  int32_t rank;                 /* 0 ≤ rank ≤ TV_MAX_RANK (rank 0 = one element)     */
  int32_t itemsize;             /* bytes per (source) element                         */
  int32_t src_dtype;            /* TV_DT_RAW, or the source TV_DT_* of a conversion   */
  int32_t dst_dtype;            /* destination TV_DT_* of a conversion                */
  uint64_t flags;               /* conversion: device address of a uint32 check word  */
} tv_copy;

/* One chunk payload to persist (save side).  The payload is the row-major bytes of
 * the box `src`/`ext` — chunkstore.py:387-392 (`np.ascontiguousarray(values[sel])
 * .tobytes()`) — and lands at byte `file_off` of output `file`. */
typedef struct tv_write_item {
  tv_array_box src;             /* source shard on `device` (or snapshot arena)       */
  int64_t ext[TV_MAX_RANK];
  int32_t rank;
  int32_t itemsize;
  int32_t file;                 /* index into the output table                        */
  int32_t device;               /* CUDA ordinal holding src                           */
  int64_t file_off;             /* payload offset inside the output                   */
} tv_write_item;

/* One output of a save: a file written atomically as <path>.partial → rename
 * (backend.py:398-403), or — when path is NULL/empty — a caller host buffer `host`
 * of `size` bytes (used for non-filesystem backends, which then receive a put). */
typedef struct tv_output {
  const char* path;
  uint64_t host;
  int64_t size;
} tv_output;

/* One contiguous byte range to fetch (restore side) — chunkstore.py:487-505
 * (`_fetch_chunk` / `_fetch_span`).  The bytes land on `device` at `direct_dst`
 * when nonzero (destination already contiguous: no staging, no kernel), otherwise in
 * device staging.  Then copies[first_copy, first_copy+n_copies) run with their
 * src.base interpreted as an OFFSET into the landed bytes (chunkstore.py:579-592,
 * load_pipeline.py:467-471, fused with the NVLink fan-out to other GPUs). */
typedef struct tv_read_item {
  int32_t input;                /* index into the input table                         */
  int32_t device;               /* reader GPU                                         */
  int64_t in_off;               /* byte offset inside the input                       */
  int64_t nbytes;
  uint64_t direct_dst;
  int32_t first_copy;
  int32_t n_copies;
} tv_read_item;

/* One input of a restore: a file path, or a caller host buffer when path is NULL. */
typedef struct tv_input {
  const char* path;
  uint64_t host;
  int64_t size;
} tv_input;

typedef struct tv_stats {
  int64_t bytes_device;         /* payload bytes moved over PCIe                      */
  int64_t bytes_storage;        /* payload bytes written to / read from outputs       */
  int64_t bytes_packed;         /* bytes produced by the box-copy kernel              */
  int64_t kernel_launches;
  int64_t dma_copies;
  int64_t files;                /* files committed (save) or opened (restore)         */
  double seconds_total;
  double seconds_kernel;        /* CUDA-event time of box-copy kernels                */
  double seconds_io;            /* storage threads: time inside pwrite/pread (summed) */
  double seconds_wait_dma;      /* storage threads: time waiting for D2H/H2D events   */
  double seconds_wait_slot;     /* producer: time waiting for a free pinned slot      */
  int64_t recycled_files;       /* save: outputs written over a recycled file (pool)  */
  int64_t zero_copy_bytes;      /* bytes DMA'd straight into / out of registered file pages */
  int64_t registered_files;     /* save: recycled files registered with CUDA by this call */
} tv_stats;

typedef struct tv_engine tv_engine;

/* ---- library --------------------------------------------------------------------- */
int tv_abi_version(void);
int tv_last_error(char* buf, size_t len);

/* ---- kernels ---------------------------------------------------------------------- */
/* Batched N-d box copy on `device`/`stream` (one launch for all copies).  Replaces the
 * numpy slicing copies of save_pipeline.py:323-324 (snapshot), chunkstore.py:392 (pack),
 * chunkstore.py:592 and load_pipeline.py:471 (unpack / assemble).  Addresses may be
 * local device, peer device (NVLink P2P / IPC) or mapped pinned host memory. */
int tv_copy_boxes(int device, const tv_copy* copies, int n, void* stream);

/* Bytes a box copy moves (sum of extents × itemsize) — for roofline accounting. */
int64_t tv_copy_bytes(const tv_copy* copies, int n);

/* Kernel timing (instrumentation for bench.py's roofline): while enabled, every box-copy
 * or cast launch of the library — tv_copy_boxes and the engine's pack / unpack / fan-out
 * launches — is bracketed by CUDA timing events on its own stream (the first recorded
 * after the job-table upload, so the window is the kernel, not the host's enqueue).
 * collect() waits for the recorded launches and returns their summed and longest
 * durations, their algorithmic HBM bytes (read + write) and their count, then resets. */
int tv_kernel_timing(int enable);
int tv_kernel_timing_collect(double* ms_total, double* ms_max, int64_t* bytes, int64_t* launches);

/* ---- engine ----------------------------------------------------------------------- */
/* Pinned host slot ring (n_slots × slot_bytes), device staging of staging_bytes on each
 * device that touches it, and n_threads storage threads. */
int tv_engine_create(int n_slots, int64_t slot_bytes, int64_t staging_bytes, int n_threads,
                     tv_engine** out);
int tv_engine_destroy(tv_engine* e);

/* Save: persist every item (ProcessArrayWriter.write_array/_put_chunk/_flush_file,
 * chunkstore.py:352-424, plus FilesystemBackend._put, backend.py:398-403).  Outputs are
 * committed (rename) when all their bytes are written.  Blocking; call from a worker
 * thread (ctypes releases the GIL). */
int tv_engine_save(tv_engine* e, const tv_write_item* items, int n_items,
                   const tv_output* outputs, int n_outputs, tv_stats* stats);
/* tv_engine_save, drawing output files from a recycle pool (`pool_dir`, may be NULL):
 * an output of N bytes claims a retired file `<pool_dir>/<N>/<name>` (rename to its
 * `.partial`) and overwrites it in place — no page allocation or zeroing for storage
 * that keeps its pages (tmpfs).  Steady-state checkpointing with retention
 * (training_manager.py:262-295: a step is retired while the next is saved).
 * pool_flags & TV_POOL_REGISTER: claimed files on a RAM-backed filesystem not registered
 * with CUDA yet are registered (map + cudaHostRegister, once per file lifetime, cached by
 * inode) up to TVGPU_REGISTER_BUDGET (default 1.0) of the save's bytes.
 * pool_flags & TV_POOL_ZERO_COPY: the contiguous items of a claimed, registered file are
 * DMA'd straight into its page-cache pages (zero-copy); everything else takes the pinned
 * slot + pwrite path. */
#define TV_POOL_REGISTER 1
#define TV_POOL_ZERO_COPY 2
int tv_engine_save_pooled(tv_engine* e, const tv_write_item* items, int n_items,
                          const tv_output* outputs, int n_outputs, const char* pool_dir,
                          int pool_flags, tv_stats* stats);

/* Restore: fetch every item once, land it on its reader GPU, run its copies
 * (ChunkReader.read_range, chunkstore.py:507-593, _execute_reads + _assemble,
 * load_pipeline.py:406-493).  Blocking. */
int tv_engine_load(tv_engine* e, const tv_read_item* items, int n_items, const tv_input* inputs,
                   int n_inputs, const tv_copy* copies, int n_copies, tv_stats* stats);

/* ---- peer access / IPC (NVLink fan-out) -------------------------------------------- */
/* Enable P2P between every ordered pair of the given CUDA ordinals (single process). */
int tv_enable_peer_access(const int* devices, int n);
/* Export / import a CUDA IPC handle (64 bytes) for a device allocation (multi-process). */
int tv_ipc_export(int device, uint64_t ptr, uint8_t handle_out[64], uint64_t* base_offset_out);
int tv_ipc_import(int device, const uint8_t handle[64], uint64_t* ptr_out);
int tv_ipc_close(int device, uint64_t ptr);

/* ---- bulk delete ------------------------------------------------------------------- */
/* Unlink n files on n_threads native threads (retention deletes of a whole checkpoint:
 * freeing tmpfs pages is per-inode kernel work; native threads keep it off the caller's
 * interpreter lock).  ok[i] = 1 if paths[i] was removed, 0 if it did not exist; any other
 * failure returns TV_ERR_IO with the first failing path (training_manager.py:262-279). */
int tv_unlink_many(const char* const* paths, int n, int n_threads, uint8_t* ok);
/* Retire files into a recycle pool instead of unlinking them: each regular file moves to
 * `<pool_dir>/<its size>/<unique name>` (same filesystem: a rename, pages kept); ok[i] as
 * tv_unlink_many.  Files that cannot be renamed there are unlinked. */
int tv_recycle_many(const char* const* paths, int n, const char* pool_dir, int n_threads,
                    uint8_t* ok);

/* Zero-copy recycle pool: map (MAP_SHARED) and register with CUDA every file of the
 * pool on a RAM-backed filesystem that is not registered yet.  A registered file keeps
 * its registration while it cycles pool -> checkpoint -> pool, and saves / restores then
 * DMA straight into / out of its page-cache pages.  No GPU: returns TV_OK, 0 bytes. */
int tv_pool_register(const char* pool_dir, int n_threads, int64_t* registered_bytes);
/* Release the registrations of, and unlink, every pool file. */
int tv_pool_drain(const char* pool_dir, int64_t* freed_bytes);
/* Registered mappings held by this process (files, bytes). */
int tv_mapping_stats(int64_t* files, int64_t* bytes);
/* Release every registered mapping (the files stay). */
int tv_mapping_release_all(void);

/* ---- roofline probes (same run as the numbers they bound) ------------------------- */
/* fio-style sequential write then read of n_threads files of file_bytes each, in
 * block_bytes pwrite/pread calls from pinned memory.  Files are removed afterwards. */
int tv_probe_storage(const char* dir, int n_threads, int64_t file_bytes, int64_t block_bytes,
                     double* write_gbps, double* read_gbps);
/* The storage probe plus a rewrite pass between write and read: the same files written
 * again without truncation (pages already allocated: the recycled-file save path). */
int tv_probe_storage_rewrite(const char* dir, int n_threads, int64_t file_bytes,
                             int64_t block_bytes, double* write_gbps, double* rewrite_gbps,
                             double* read_gbps);
/* The same storage probe while a DMA thread keeps `device`'s copy engine busy for the
 * whole window (D2H during the writes, H2D during the reads): the contended rates of a
 * copy-through-pinned pipeline, whose DMA and page-cache copies share host memory. */
int tv_probe_storage_dma(const char* dir, int n_threads, int64_t file_bytes, int64_t block_bytes,
                         int device, double* write_gbps, double* read_gbps, double* d2h_gbps,
                         double* h2d_gbps);
/* Pinned D2H and H2D copy bandwidth of `device` over `bytes` (best of `reps`). */
int tv_probe_pcie(int device, int64_t bytes, int reps, double* d2h_gbps, double* h2d_gbps);

#ifdef __cplusplus
}
#endif
#endif /* TVGPU_H */
