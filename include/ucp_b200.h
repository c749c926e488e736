/*
 * ucp_b200.h -- C ABI of libucp_b200.so, the sm_100a data-movement engine
 * behind the Universal Checkpointing reshard hot path.
 *
 * The reference (/root/reference/pkg/src/ucp) is pure Python + numpy and has no
 * FFI; the entry points below are what its per-element work would bind to.
 * Each one cites the reference function whose inner loop it replaces:
 *
 *   ucp_convert_gather  <- union()            ucp/convert.py:221-308
 *                          _collapse_dp()      ucp/convert.py:137-193
 *                          strip_pad()         ucp/convert.py:115-129
 *                          _union_hy()         ucp/convert.py:196-218
 *   ucp_load_scatter    <- extract_fragment()  ucp/parallel.py:373-411
 *                          partial_noise()     ucp/parallel.py:340-370
 *                          cast()              ucp/tensor.py:208-223 (load epilogue, ucp/load.py:204-205)
 *   ucp_gen_state       <- hash_unit()/gen_tensor()  ucp/tensor.py:162-184, init_state() ucp/models.py:230-244
 *
 * Work is described by a host-compiled table of 2-D strided "runs" (see
 * DESIGN.md §3). A run moves rows x cols f32 elements from n_src sources to
 * n_dst destinations with one element-wise op. Sources are laid out
 * group-major: source (g, k) is the k-th replica of group g; replicas must be
 * bit-identical to replica 0 of their group (strict replica check), groups
 * are averaged in f64 in ascending order (MEAN). The table is executed by a
 * grid of one CTA per tile; tiles never straddle runs. Runs are sorted by
 * kernel class; each run carries a ucp_runtile (its tile size and count),
 * ucp_runtile_scan turns the counts into per-class tile offsets on the
 * device (a block-wide scan built from warp shuffles), and each CTA finds
 * its run with a warp-cooperative 32-ary search over those offsets, so no
 * per-tile table exists in memory.
 *
 * Conventions: all pointers are device pointers, all calls are
 * stream-ordered and reentrant (no global state besides the caller's status
 * word). Return value is 0 or a negative UCP_E* code for argument / launch
 * errors. Data-dependent failures (replica mismatch, nonzero pad) are
 * reported asynchronously through ucp_status, read by the caller after the
 * stream synchronises.
 */
#ifndef UCP_B200_H
#define UCP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UCP_ABI_VERSION 3

/* status / return codes (mirrored in paper_2406_18820_b200/_errors.py) */
#define UCP_OK 0
#define UCP_EREPLICA (-1)  /* ReplicateMismatchError */
#define UCP_EPAD (-2)      /* PaddingError */
#define UCP_EINVAL (-10)   /* bad argument / descriptor */
#define UCP_ECUDA (-11)    /* CUDA launch or runtime error */

/* run ops */
#define UCP_OP_COPY 0      /* dst = src(g=0,k=0); replicas verified */
#define UCP_OP_MEAN 1      /* dst = f32(sum_g f64(src(g,0)) / groups); replicas verified */
#define UCP_OP_NOISE 2     /* dst = partial_noise(src, tp_rank, tp) */
#define UCP_OP_ZERO 3      /* dst = +0.0 (ZeRO re-pad); n_src == 0 */
#define UCP_OP_CHECKZERO 4 /* verify src bits == 0 (pad strip); n_dst == 0 */

/* destination dtypes (UCPT dtype codes, ucp/tensor.py:43-59) */
#define UCP_DT_F32 0
#define UCP_DT_F16 1
#define UCP_DT_BF16 2

/* kernel classes: runs are sorted by class, each class runs its own kernel */
#define UCP_CLASS_VEC_F32 0   /* COPY, UCP_RUN_VEC, f32 destinations */
#define UCP_CLASS_VEC_BF16 1  /* COPY, UCP_RUN_VEC, bf16 destinations */
#define UCP_CLASS_VEC_F16 2   /* COPY, UCP_RUN_VEC, f16 destinations */
#define UCP_CLASS_GENERAL 3   /* COPY runs whose pieces do not share one 16-B phase (realigned) */
#define UCP_CLASS_OPS 4       /* MEAN / NOISE / ZERO / CHECKZERO (move tables only) */
#define UCP_NCLASS 5

/* run flags */
#define UCP_RUN_VEC 1u       /* every src/dst row start shares one 16-B phase */
#define UCP_RUN_ROWSPLIT 2u  /* tiles cut columns of single rows */

typedef struct ucp_run {
  uint64_t src;        /* byte offset of source (0,0) from src_base, replica (0,0) */
  uint64_t dst;        /* byte offset of destination 0's (0,0) from dst_base */
  uint32_t src_pitch;  /* elements between source rows */
  uint32_t dst_pitch;  /* elements between destination rows */
  uint32_t rows;
  uint32_t cols;       /* elements per row; rows*cols < 2^32 */
  uint32_t aux;        /* index in aux[] of extra offsets: sources 1..n_src-1, then dsts 1..n_dst-1 */
  uint16_t n_src;      /* groups * replicas-per-group (0 for ZERO) */
  uint16_t n_dst;      /* fan-out (0 for CHECKZERO) */
  uint16_t groups;     /* averaged groups (MEAN), else 1 */
  uint8_t op;          /* UCP_OP_* */
  uint8_t dtype;       /* UCP_DT_* of destinations; sources are always f32 */
  uint16_t tp_rank;    /* NOISE */
  uint16_t tp;         /* NOISE */
  uint32_t tag;        /* caller's unit id, echoed in errors */
  uint32_t flags;      /* UCP_RUN_* */
  uint32_t pad_;
} ucp_run;             /* 64 bytes */

/*
 * Fused reshard run (convert + load in one pass): rows x cols
 * f32 elements read from n_src bit-identical replicas (strict check), written
 * once to the atomic tensor (f32, atom_pitch; skipped when atom == UINT64_MAX)
 * and fanned out to n_dst target fragments (dtype, dst_pitch). The atomic
 * bytes are never read back: the load half consumes them from registers.
 */
typedef struct ucp_xrun {
  uint64_t src;        /* byte offset from src_base of replica 0's (0,0) */
  uint64_t atom;       /* byte offset from atom_base, or UINT64_MAX */
  uint64_t dst;        /* byte offset from dst_base of target 0's (0,0) */
  uint32_t src_pitch;  /* elements */
  uint32_t atom_pitch;
  uint32_t dst_pitch;
  uint32_t rows;
  uint32_t cols;
  uint32_t aux;        /* sources 1..n_src-1, then targets 1..n_dst-1 */
  uint16_t n_src;
  uint16_t n_dst;
  uint8_t dtype;       /* UCP_DT_* of the targets */
  uint8_t pad0_;
  uint16_t pad1_;
  uint32_t tag;
  uint32_t flags;      /* UCP_RUN_VEC (vector classes) or clear (GENERAL); UCP_RUN_ROWSPLIT */
} ucp_xrun;            /* 64 bytes */

/* Per-run tiling, parallel to the run array. The host fills per / tpr /
 * ntiles; ucp_runtile_scan fills first. Tile k of a run covers
 *   default:          rows [k*per, min((k+1)*per, rows)), all columns
 *   UCP_RUN_ROWSPLIT: row k / tpr, columns [(k % tpr)*per, +per) clipped. */
typedef struct ucp_runtile {
  uint32_t first;      /* exclusive prefix of ntiles within the run's class */
  uint32_t per;        /* rows per tile, or columns per tile (ROWSPLIT) */
  uint32_t tpr;        /* tiles per row (ROWSPLIT), else 0 */
  uint32_t ntiles;
} ucp_runtile;         /* 16 bytes */

/* A tile as one CTA derives it (device-internal; not stored anywhere). */
typedef struct ucp_tile {
  uint32_t run;
  uint32_t row0;
  uint32_t col0;
  uint32_t count;      /* rows (default) or cols (UCP_RUN_ROWSPLIT) */
} ucp_tile;            /* 16 bytes */

typedef struct ucp_status {
  /* min over failures of (run index << 32 | element index in run); ~0 = ok */
  unsigned long long first;
  unsigned long long n_bad;  /* failing (warp, segment) reports, for stats */
} ucp_status;

/* Version of this ABI (UCP_ABI_VERSION). */
int ucp_version(void);

/* Build provenance: "UCP_BUILD_ID:" + the first 32 hex digits of
 * sha256(csrc/ucp_b200.cu || include/ucp_b200.h), baked in by the build
 * (paper_2406_18820_b200/_build.py); the loader refuses a library whose id
 * differs from the sources next to it. */
const char* ucp_build_id(void);

/* Reset a device status word to "no failure" (stream-ordered). */
int ucp_status_reset(ucp_status* status, void* stream);

/*
 * Fill ucp_runtile.first: per class, the exclusive prefix sum of ntiles over
 * the class's runs (one CTA per class, warp-shuffle scans). Call once after
 * uploading a table; class_info is a HOST array of 2*UCP_NCLASS int64:
 * tiles per class, then runs per class (runs sorted by class).
 */
int ucp_runtile_scan(ucp_runtile* rt, const int64_t* class_info, void* stream);

/*
 * Consolidate fragments into atomic tensors (union). One launch covers any
 * number of (param, kind) units. src_base: base of the source-fragment arena;
 * dst_base: base of the atomic arena. aux: uint64 byte offsets. runs sorted by
 * class, rt: their scanned ucp_runtile array (device); class_info: HOST array
 * of 2*UCP_NCLASS int64 (tiles per class, then runs per class).
 */
int ucp_convert_gather(const ucp_run* runs, int64_t n_runs, const uint64_t* aux,
                       const ucp_runtile* rt, const int64_t* class_info, const void* src_base,
                       void* dst_base, ucp_status* status, void* stream);

/*
 * Slice atomic tensors into target fragments (extract_fragment + re-pad +
 * partial noise + weight cast), fanning each read out to n_dst replicas.
 */
int ucp_load_scatter(const ucp_run* runs, int64_t n_runs, const uint64_t* aux,
                     const ucp_runtile* rt, const int64_t* class_info, const void* src_base,
                     void* dst_base, ucp_status* status, void* stream);

/*
 * Deterministic generator: out[i] = stream value start+i of stream `base`
 * (stream_base(seed, name, tag) computed on the host), |.| if abs_flag.
 * Bit-exact with ucp/tensor.py:162-171.
 */
int ucp_gen_state(uint64_t base, uint64_t start, uint64_t count, int abs_flag, float* out,
                  void* stream);

/*
 * Fused convert + load (the in-memory resume() path, ucp/load.py:276-281):
 * class_info as for ucp_convert_gather, runs sorted by class. Classes
 * VEC_F32 / VEC_BF16 / VEC_F16 hold vector runs (UCP_RUN_VEC: one shared 16-B
 * phase) of one target dtype each; for fused tables the GENERAL slot holds
 * phase-mismatched cells (UCP_RUN_VEC clear, any target dtype), realigned in
 * registers at vector width (kernel reshard_fused_realign).
 */
int ucp_reshard_fused(const ucp_xrun* runs, int64_t n_runs, const uint64_t* aux,
                      const ucp_runtile* rt, const int64_t* class_info, const void* src_base,
                      void* atom_base, void* dst_base, ucp_status* status, void* stream);

/*
 * One bias-corrected Adam step of the reference's toy trainer, in place,
 * bit-exact with ucp/models.py:265-293 (f64 elementwise, fixed operation
 * order, RNE to f32): g = hash_unit(grad_base, start + i) (ucp/models.py:247-253),
 *   m' = b1*m + (1-b1)*g ; v' = b2*v + ((1-b2)*g)*g
 *   w' = w - (lr*(m'/bc1)) / (sqrt(v'/bc2) + eps)
 * bc1/bc2 and 1-b1/1-b2 are computed by the caller exactly as the
 * reference does (plain repeated multiplication, _pow_seq).
 */
int ucp_adam_step(float* w, float* m, float* v, uint64_t count, uint64_t grad_base,
                  uint64_t start, double b1, double one_minus_b1, double b2,
                  double one_minus_b2, double bc1, double bc2, double lr, double eps,
                  void* stream);

/* Byte-compare two device buffers; *mismatch (device) receives the first
 * differing byte index or ~0. Used by the checker paths of the bench. */
int ucp_compare(const void* a, const void* b, uint64_t nbytes, unsigned long long* mismatch,
                void* stream);

/*
 * Peer memory for the rank-homed load (north_star item 3): target fragments
 * whose home GPU is not the param owner are written by ucp_reshard_fused /
 * ucp_load_scatter straight into the home GPU's receive buffer through a
 * CUDA IPC mapping (NVLink / NVSwitch stores, overlapped with the HBM work
 * tile by tile). Buffers are cudaMalloc'ed here so the IPC handle covers the
 * allocation exactly.
 */
typedef struct ucp_ipc_handle {
  unsigned char bytes[64]; /* cudaIpcMemHandle_t */
} ucp_ipc_handle;

int ucp_dev_alloc(uint64_t nbytes, void** ptr);
int ucp_dev_free(void* ptr);
int ucp_ipc_export(const void* dev_ptr, ucp_ipc_handle* out);
/* Map a peer's buffer into this process (peer access enabled lazily). */
int ucp_ipc_open(const ucp_ipc_handle* handle, void** mapped);
int ucp_ipc_close(void* mapped);

/* Synchronous device->host copy of n bytes (error-path diagnostics: reading
 * the replicas behind a failing run to name them in the exception). */
int ucp_peek(const void* device_src, void* host_dst, uint64_t nbytes);

#ifdef __cplusplus
}
#endif

#endif /* UCP_B200_H */
