/*
 * sbnet.h — C ABI of the B200-native (sm_100a) SBNet sparse-block hot path.
 *
 * The reference (`blockconv`, /root/reference/pkg/src/blockconv) is a pure-Python
 * package; its "plugin surface" is the Python function API exported from
 * `__init__.py:9-26`.  This header is the native boundary that sits UNDER the Python
 * mirror of that API (paper_1801_02108_b200/*.py).  Each entry point below names the
 * reference function it replaces.  Conventions:
 *
 *  - plain device pointers and sizes; no torch types.  All tensors are contiguous,
 *    activations NHWC (logical (n, h, w, c), reference `tensor.py:43-49`), masks uint8
 *    (n, h, w), block index lists int32 (cap, 3) rows (frame, block_y, block_x) in
 *    ascending order plus a device-resident int32 count.
 *  - the caller owns every buffer, including workspaces; the library never allocates
 *    device memory.  `dst` / `out` arguments are mutated in place (the Python layer
 *    clones first to keep the reference's functional semantics, `blocks.py:134`).
 *  - every call is asynchronous and stream-ordered on `stream` (a cudaStream_t).  The
 *    only data-dependent quantity, the active block count, stays on the device: kernels
 *    read `*count` and run a persistent grid sized for `cap` rows, so no host sync is
 *    needed between reduce_mask and the consumers.
 *  - return 0 on success, a negative SBN_ERR_* code otherwise; sbn_last_error() returns
 *    a message (thread-local).  The Python layer maps codes onto the reference's
 *    exception classes (`errors.py:4-35`).
 */
#ifndef SBNET_H_
#define SBNET_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* sbn_stream_t; /* cudaStream_t */

enum sbn_status {
  SBN_OK = 0,
  SBN_ERR_INVALID = -1,     /* bad argument (-> ValueError / GeometryError) */
  SBN_ERR_SHAPE = -2,       /* inconsistent dims (-> ShapeMismatchError) */
  SBN_ERR_UNSUPPORTED = -3, /* dtype/config not implemented (-> UnsupportedConfigError) */
  SBN_ERR_WORKSPACE = -4,   /* workspace too small */
  SBN_ERR_CUDA = -5         /* launch / runtime error */
};

enum sbn_dtype { SBN_F32 = 0, SBN_F64 = 1, SBN_BF16 = 2 };
enum sbn_pool { SBN_POOL_MAX = 0, SBN_POOL_AVG = 1 };
enum sbn_algo { SBN_ALGO_AUTO = 0, SBN_ALGO_SIMT = 1, SBN_ALGO_TCGEN05 = 2 };

/* Overlap-save tiling of one layer; the fields of the reference BlockSpec
 * (`tiling.py:47-61`) as computed by `compute_block_spec` (`tiling.py:64-99`). */
typedef struct sbn_geometry {
  int32_t n, h, w;     /* input frames and spatial extent */
  int32_t bh, bw;      /* block_size (input window incl. halo) */
  int32_t sy, sx;      /* in_stride = block - overlap */
  int32_t oy, ox;      /* grid_origin (<= 0) */
  int32_t gy, gx;      /* grid_count */
  int32_t obh, obw;    /* out_block_size (= output stride) */
  int32_t oh, ow;      /* out_size of the dense conv */
} sbn_geometry;

/* Inference-mode bottleneck unit (reference ResidualUnitParams, `layers.py:85-114`).
 * Filters HWIO (kh, kw, cin, cout) in the activation dtype; biases (cout) in the
 * activation dtype; BN folded to per-channel scale/shift (`ops.py:213-216`) in the
 * compute dtype (float for F32/BF16, double for F64). */
typedef struct sbn_unit_params {
  const void* w1; const void* b1;   /* 1x1, c -> m */
  const void* w2; const void* b2;   /* 3x3, m -> m */
  const void* w3; const void* b3;   /* 1x1, m -> c */
  const void* bn1_scale; const void* bn1_shift;
  const void* bn2_scale; const void* bn2_shift;
  const void* bn3_scale; const void* bn3_shift;
  /* optional: pre-packed tensor-core image from sbn_residual_unit_pack (NULL: the call
   * packs into its workspace first, one extra launch) */
  const void* tc_packed;
  /* identity of tc_packed: the byte count sbn_residual_unit_packed_bytes and the
   * variant sbn_residual_unit_packed_variant reported for the geometry it was packed
   * for.  The image layout depends on the variant the geometry selects (block size,
   * batch size); a call whose variant needs another image rejects it with
   * SBN_ERR_INVALID instead of reading a foreign layout. */
  size_t tc_packed_bytes;
  int tc_packed_variant;
} sbn_unit_params;

const char* sbn_version(void);
const char* sbn_last_error(void);
int sbn_device_sm_count(int device);

/* reduce_mask (`tiling.py:138-160`): pool each block's input window of `mask`
 * (zero outside the image) and emit active blocks in ascending (n, by, bx) order.
 * MAX: any pixel set.  AVG: count/(bh*bw) >= threshold - 1e-12 in float64.
 * idx: int32 (n*gy*gx, 3) capacity; count: one int32.  ws: sbn_reduce_mask_workspace
 * bytes, ZEROED ONCE by the caller at allocation (the kernel leaves it zeroed). */
size_t sbn_reduce_mask_workspace(const sbn_geometry* g);
int sbn_reduce_mask(const uint8_t* mask, const sbn_geometry* g, int pool, double threshold,
                    int32_t* idx, int32_t* count, void* ws, size_t ws_bytes, sbn_stream_t stream);

/* downsample_mask (`tiling.py:163-174`): max-pool window = stride = factor, ceil dims. */
int sbn_downsample_mask(const uint8_t* in, int n, int h, int w, int factor, uint8_t* out,
                        sbn_stream_t stream);

/* gather / gather_transpose (`blocks.py:57-94`): out is (cap, bh, bw, c) NHWC or
 * (cap, c, bh, bw) when transpose != 0; rows >= *count are left untouched. */
int sbn_gather(const void* x, int dtype, int c, const sbn_geometry* g, const int32_t* idx,
               const int32_t* count, int cap, int transpose, void* out, sbn_stream_t stream);

/* in_bounds_map (`blocks.py:97-112`): uint8 (cap, bh, bw). */
int sbn_in_bounds(const sbn_geometry* g, const int32_t* idx, const int32_t* count, int cap,
                  uint8_t* out, sbn_stream_t stream);

/* scatter / scatter_add / scatter_transpose (`blocks.py:115-159`): write (add != 0:
 * accumulate) each (obh, obw, c) block — (c, obh, obw) when transpose != 0 — into
 * dst (n, oh, ow, c) at (by*obh, bx*obw), clipped to (oh, ow). */
int sbn_scatter(const void* blocks, int dtype, int c, const sbn_geometry* g, const int32_t* idx,
                const int32_t* count, int cap, int add, int transpose, void* dst,
                sbn_stream_t stream);

/* gather_grad (`blocks.py:162-188`): adjoint of gather.  dx (n, h, w, c) is fully written:
 * each element is the sum of the covering active blocks' values of gblk (cap, bh, bw, c)
 * in ascending block order starting from zero (the reference's `+=` sequence: bit-exact
 * for F32/F64; BF16 accumulates in fp32).  ws: sbn_gather_grad_workspace bytes (block
 * table), scratch.  scatter_grad (`blocks.py:191-204`) needs no entry of its own: it is
 * sbn_gather over the output grid (h, w = out size, block = stride = out block, origin 0). */
size_t sbn_gather_grad_workspace(const sbn_geometry* g);
int sbn_gather_grad(const void* gblk, int dtype, int c, const sbn_geometry* g, const int32_t* idx,
                    const int32_t* count, int cap, void* dx, void* ws, size_t ws_bytes,
                    sbn_stream_t stream);

/* Copy each active block's region between two frames of identical shape at the same
 * coordinates: region 0 = the input window clipped to the image, region 1 = the clipped
 * output window, region 2 = the union of the active input windows (every pixel once: the
 * overlap rims an earlier active neighbour covers are skipped; falls back to 0 when the
 * overlap exceeds half the block).  Either pointer may be pinned host memory (UVA): this moves exactly the
 * bytes a sparse layer reads / writes between a host-resident frame and its device
 * staging copy (the host-frame path of sparse_residual_unit).  No reference counterpart:
 * the reference operates on host arrays in place of this transfer. */
int sbn_copy_block_regions(const void* src, void* dst, int dtype, int c, const sbn_geometry* g,
                           const int32_t* idx, const int32_t* count, int cap, int region,
                           sbn_stream_t stream);
/* The same window regions (0 input windows, 1 output windows) between a CHANNELS_FIRST
 * (n, c, h, w) tensor and a CHANNELS_LAST one of the same logical dims: dir 0 copies
 * NCHW src -> NHWC dst, dir 1 NHWC src -> NCHW dst (bit-exact transposing copies), so
 * CHANNELS_FIRST callers reach the NHWC kernels at the cost of the active windows only. */
int sbn_copy_block_regions_t(const void* src, void* dst, int dtype, int c, const sbn_geometry* g,
                             const int32_t* idx, const int32_t* count, int cap, int region, int dir,
                             sbn_stream_t stream);

/* Dense k x k convolution (k = 1, 3, 5; stride <= min(k, 3)), bias fused (bf16, tcgen05
 * implicit GEMM fed by strided 4-D TMA boxes): the stage-transition projection of run_stage
 * (reference `layers.py:316-318`: conv2d_direct + bias).  x (n, h, w, cin) NHWC; out
 * (n, oh, ow, cout); padding (ph, pw) zero-fill; packed: sbn_dense_conv_packed_bytes, from
 * sbn_dense_conv_pack of the HWIO weights; bias: cout floats.  Channel counts need only be
 * multiples of 8 (16-byte pixel rows): K and N are padded to the 16-wide UMMA granule inside
 * (TMA zero-fills the K padding, the packed image holds zero rows/columns, the epilogue drops
 * the N padding); instantiated shapes are reported by sbn_dense_conv_supported. */
int sbn_dense_conv_supported(int dtype, int cin, int cout, int kh, int kw, int sh, int sw);
size_t sbn_dense_conv_packed_bytes(int cin, int cout, int k);
int sbn_dense_conv_pack(const void* w, int cin, int cout, int k, void* packed, sbn_stream_t stream);
int sbn_dense_conv(const void* x, int n, int h, int w, int cin, int cout, int k, int sh, int sw, int ph,
                   int pw, int oh, int ow, const void* packed, const float* bias, void* out, sbn_stream_t stream);

/* Fused sparse_conv2d body (`layers.py:27-47` after reduce_mask): gather -> valid
 * conv (kh, kw, stride sh, sw) -> (+bias) -> scatter into dst (n, oh, ow, cout), all in
 * one kernel; the block stack never touches HBM.  w: HWIO; bias nullable.
 * w_packed: optional tensor-core weight image (sbn_sparse_conv_pack); when NULL on the
 * tcgen05 path the call packs into ws (sbn_sparse_conv_packed_bytes bytes) first. */
int sbn_sparse_conv(const void* x, int dtype, int cin, int cout, int kh, int kw, int sh, int sw,
                    const sbn_geometry* g, const void* w, const void* bias, const void* w_packed,
                    const int32_t* idx, const int32_t* count, int cap, void* dst, void* ws,
                    size_t ws_bytes, int algo, sbn_stream_t stream);
/* sparse_conv2d straight from the mask (reference `layers.py:27-47`, MAX pool with the
 * default threshold): ONE kernel where the tcgen05 kernels allow it — the 3x3 row-shift
 * conv with >= 64 candidates per CTA, and the tap-GEMM conv on grids of at most four
 * (candidate block, sub-tile) units per CTA slot — each CTA tests its own candidates' windows and
 * convolves the active ones (unordered; the output does not depend on the order);
 * otherwise reduce_mask + sparse_conv.  sync_ws: sbn_sparse_conv_masked_sync_bytes, zeroed
 * ONCE by the caller and kept between calls (launch epoch, counters, reduce_mask words at
 * fixed offsets: calls of any geometry may share it); ws: ..._workspace bytes of scratch. */
size_t sbn_sparse_conv_masked_sync_bytes(const sbn_geometry* g);
size_t sbn_sparse_conv_masked_workspace(int dtype, int cin, int cout, int kh, int kw, int sh, int sw,
                                        const sbn_geometry* g);
int sbn_sparse_conv_masked(const void* x, const uint8_t* mask, int dtype, int cin, int cout, int kh, int kw,
                           int sh, int sw, const sbn_geometry* g, const void* w, const void* bias,
                           const void* w_packed, void* dst, void* sync_ws, size_t sync_bytes, void* ws,
                           size_t ws_bytes, int algo, sbn_stream_t stream);
size_t sbn_sparse_conv_packed_bytes(int dtype, int cin, int cout, int kh, int kw, int sh, int sw,
                                    const sbn_geometry* g);
int sbn_sparse_conv_pack(const void* w, int dtype, int cin, int cout, int kh, int kw, int sh,
                         int sw, const sbn_geometry* g, void* packed, sbn_stream_t stream);

/* Fused sparse_residual_unit body (`layers.py:203-229` after reduce_mask): gather ->
 * bottleneck branch (`_unit_branch`, `layers.py:137-179`) -> scatter_add onto out.
 * out must hold x's values on entry (out == x is allowed: in-place, as the paper's
 * fused scatter-add).  halo >= 0 as in the reference; pre_act selects the chain. */
size_t sbn_residual_unit_workspace(int dtype, int c, int m, const sbn_geometry* g, int halo,
                                   int algo);
int sbn_residual_unit(const void* x, int dtype, int c, int m, const sbn_geometry* g, int halo,
                      int pre_act, const sbn_unit_params* p, const int32_t* idx,
                      const int32_t* count, int cap, void* out, void* ws, size_t ws_bytes,
                      int algo, sbn_stream_t stream);

/* Tensor-core weight image: W1/W2/W3 transposed into the kernel's shared-memory operand
 * layout plus the folded BN/bias vectors, built once per parameter set and block size
 * and bulk-copied by every CTA.  bytes == 0: the tcgen05 path does not apply. */
size_t sbn_residual_unit_packed_bytes(int dtype, int c, int m, const sbn_geometry* g, int halo,
                                      int pre_act);
/* Which tensor-core unit (and so which packed image layout) a call with this geometry
 * runs: 1 = fused single kernel (unit_tc.cu), 2 = wide three-launch unit (unit_wide.cu),
 * 0 = none (SIMT).  Depends on the candidate count n*gy*gx, not only the block size. */
int sbn_residual_unit_packed_variant(int dtype, int c, int m, const sbn_geometry* g, int halo,
                                     int pre_act);
int sbn_residual_unit_pack(const sbn_unit_params* p, int dtype, int c, int m,
                           const sbn_geometry* g, int halo, int pre_act, void* packed,
                           sbn_stream_t stream);

/* The whole sparse_residual_unit (`layers.py:203-229`): mask -> active blocks (MAX pool
 * over each block's input window) -> fused unit -> scatter-add into out.  On the
 * tcgen05 path this is ONE kernel: the mask reduction is fused in front of the unit and
 * produces an unordered active list (blocks write disjoint windows, so the result does
 * not depend on the order).  sync_ws: sbn_sparse_residual_unit_sync_bytes, zeroed ONCE by
 * the caller and left zeroed by every call (barrier / look-back words at fixed offsets);
 * ws: sbn_sparse_residual_unit_workspace bytes, zeroed ONCE by the caller and kept between
 * calls (it carries the launch epoch and the tagged block-list entries; a new zeroed ws
 * simply restarts the epoch).  Kernels are launched with programmatic dependent launch: the
 * tcgen05 kernel reads the packed weights and tests its first round of mask candidates
 * before griddepcontrol.wait, i.e. possibly while the previous kernel on the stream is
 * still running — `mask` (like the packed image) must not be written by a kernel that
 * triggers its dependents early (no kernel of this library that writes masks does). */
size_t sbn_sparse_residual_unit_sync_bytes(const sbn_geometry* g);
size_t sbn_sparse_residual_unit_workspace(int dtype, int c, int m, const sbn_geometry* g, int halo,
                                          int algo);
int sbn_sparse_residual_unit(const void* x, const uint8_t* mask, int dtype, int c, int m,
                             const sbn_geometry* g, int halo, int pre_act,
                             const sbn_unit_params* p, void* out, void* sync_ws, size_t sync_bytes,
                             void* ws, size_t ws_bytes, int algo, sbn_stream_t stream);

/* Which algorithm `algo=AUTO` would pick (SBN_ALGO_SIMT / SBN_ALGO_TCGEN05). */
int sbn_residual_unit_algo(int dtype, int c, int m, const sbn_geometry* g, int halo, int pre_act);
int sbn_sparse_conv_algo(int dtype, int cin, int cout, int kh, int kw, int sh, int sw,
                         const sbn_geometry* g);

/* Diagnostics: tensor-core descriptor self test.  d[128 x 32] (fp32) =
 * a[shift:shift+128, 0:32] @ b[0:32, 0:32]^T with a (rows x 32) and b (32 x 32) bf16
 * row-major, staged in the plane layout with plane stride rows*16 + plane_pad bytes. */
int sbn_selftest_umma(const void* a, const void* b, int rows, int shift, int plane_pad, float* d,
                      sbn_stream_t stream);

/* Diagnostics: when buf != NULL the fused kernels record %globaltimer at phase
 * boundaries into buf[cta * 16 + phase] (buf: device memory, grid * 16 slots). */
int sbn_debug_set_trace(unsigned long long* buf);

/* Diagnostics: kernel-variant switches (returns the previous value).
 * SBN_DEBUG_NO_PAIR: run the single-CTA tcgen05 unit instead of the CTA-pair variant.
 * SBN_DEBUG_CONV_SINGLE_BUFFER: run the single-buffered tcgen05 conv kernel.
 * SBN_DEBUG_FORCE_WIDE: run the three-launch wide tcgen05 unit even where the single-kernel
 * unit applies.
 * SBN_DEBUG_FORCE_FUSED: run the single-kernel unit wherever it is supported (ignores the
 * candidate-count switch-over to the wide unit).
 * SBN_DEBUG_CONV_TMA: run sparse convs on the strided-TMA tap-GEMM kernel even where the
 * single-window kernel applies.
 * SBN_DEBUG_CONV_PAIR: run 16x16-block 3x3 sparse convs on the CTA-pair (cta_group::2,
 * M = 256) kernel with streamed weights.
 * SBN_DEBUG_CONV_NO_RESIDENT: do not use the resident-weight CTA-pair conv (16x16 blocks,
 * 128 -> 128 channels); the single-CTA double-buffered kernel runs instead.
 * SBN_DEBUG_NO_EARLY_MASK: the mask-fused tcgen05 unit tests its first round of candidates
 * after griddepcontrol.wait instead of before it.
 * SBN_DEBUG_ROW_REDUCE_MASK: reduce_mask on the one-block-row-per-CTA kernel even where the
 * ranges kernel (several block rows per CTA) applies.
 * SBN_DEBUG_CONV_RES_ONE_LAUNCH: sparse_conv2d from the mask on the resident-weight CTA pair
 * as ONE launch (mask test + global list inside the conv) instead of reduce_mask + the
 * pair's list mode.
 * SBN_DEBUG_NO_MASK_PDL: launch the cluster reduce_mask without programmatic dependent
 * launch and keep the resident pair conv from triggering its dependents early.
 * SBN_DEBUG_TMA_GLOBAL_LIST: sparse_conv2d from the mask on the tap-GEMM conv as one launch
 * with a global block list for any window size (default: windows of 128..512 pixels). */
enum { SBN_DEBUG_NO_PAIR = 1, SBN_DEBUG_CONV_SINGLE_BUFFER = 2, SBN_DEBUG_FORCE_WIDE = 4, SBN_DEBUG_FORCE_FUSED = 8,
       SBN_DEBUG_CONV_TMA = 16, SBN_DEBUG_CONV_PAIR = 32, SBN_DEBUG_CONV_NO_RESIDENT = 2048,
       SBN_DEBUG_NO_EARLY_MASK = 4096, SBN_DEBUG_ROW_REDUCE_MASK = 8192,
       SBN_DEBUG_CONV_RES_ONE_LAUNCH = 16384, SBN_DEBUG_NO_MASK_PDL = 32768,
       SBN_DEBUG_TMA_GLOBAL_LIST = 65536 };
int sbn_debug_set_flags(int flags);
/* Diagnostics: occupancy the last tcgen05 unit launch computed (0: CTAs/SM of the
 * single-CTA kernel, 1: co-resident clusters of the CTA-pair kernel). */
int sbn_debug_last_occupancy(int which);

/* Number of kernels the library has launched since load (for the bench's
 * gpu_launches claim). */
uint64_t sbn_launch_count(void);

/* Convolution gradients (training path; reference `conv2d_grads_nhwc`, `ops.py:167-197`) of
 * a direct NHWC convolution x (n, h, w, cin) * W (kh, kw, cin, cout), stride (sh, sw),
 * zero padding (ph, pw), for an upstream gradient g (n, oh, ow, cout):
 *   sbn_conv_grad_input:  dx (n, h, w, cin) = sum over taps of g . W[i, j]^T (overwritten)
 *   sbn_conv_grad_weight: dw (kh, kw, cin, cout) and, when db != NULL, db (cout); the sums
 *     over output positions are deterministic (fixed segments reduced in order), through a
 *     caller workspace of sbn_conv_grad_weight_workspace bytes.
 * F32 / F64 / BF16 (accumulated in float / double / float). */
int sbn_conv_grad_input(const void* g, int dtype, int n, int h, int w, int cin, int oh, int ow, int cout,
                        const void* wt, int kh, int kw, int sh, int sw, int ph, int pw, void* dx,
                        sbn_stream_t stream);
size_t sbn_conv_grad_weight_workspace(int dtype, int n, int oh, int ow, int cin, int cout, int kh, int kw);
int sbn_conv_grad_weight(const void* x, const void* g, int dtype, int n, int h, int w, int cin, int oh,
                         int ow, int cout, int kh, int kw, int sh, int sw, int ph, int pw, void* dw,
                         void* db, void* ws, size_t ws_bytes, sbn_stream_t stream);

/* Training-path forward pieces (the unit backward's recomputation; F32 / F64):
 *   sbn_conv_forward: y (n, oh, ow, cout) = direct NHWC convolution of x with W (kh, kw, cin,
 *     cout) + bias (may be NULL), taps accumulated in order (reference `conv2d_nhwc`,
 *     `ops.py:145-164`);
 *   sbn_bn_relu: pre = x * scale + shift (per channel, rounded multiply then add; pre may be
 *     NULL), post = relu(pre) * valid (valid: one value per pixel = count / c, or NULL)
 *     (reference `ops.py:213-216`, `:233-234`);
 *   sbn_bn_relu_grad: out = g * valid * (pre > 0) * scale (the adjoint of sbn_bn_relu);
 *   sbn_add: out = a + b (elementwise). */
int sbn_conv_forward(const void* x, int dtype, int n, int h, int w, int cin, int oh, int ow, int cout,
                     const void* wt, int kh, int kw, int sh, int sw, int ph, int pw, const void* bias, void* y,
                     sbn_stream_t stream);
int sbn_bn_relu(const void* x, int dtype, long count, int c, const void* scale, const void* shift, const void* valid,
                void* pre, void* post, sbn_stream_t stream);
int sbn_bn_relu_grad(const void* g, const void* pre, int dtype, long count, int c, const void* scale,
                     const void* valid, void* out, sbn_stream_t stream);
int sbn_add(const void* a, const void* b, int dtype, long count, void* out, sbn_stream_t stream);

/* Train-mode batch norm over gathered blocks (reference `sparse_batch_norm`, TRAIN_STATS,
 * `layers.py:68-82`): x is (rows, c); per-channel mean and population variance (deterministic
 * segmented sums, in the dtype's accumulation type) are written to mean / var (c values of the
 * accumulation type: float for F32, double for F64) and
 * out = (x - mean) * (gamma / sqrt(var + eps)) + beta.  F32 / F64. */
size_t sbn_bn_train_workspace(int dtype, long rows, int c);
int sbn_bn_train(const void* x, int dtype, long rows, int c, const void* gamma, const void* beta, double eps,
                 void* out, void* mean, void* var, void* ws, size_t ws_bytes, sbn_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SBNET_H_ */
