/*
 * rsgrad.h — C ABI of the B200 (sm_100a) resampling-layer library.
 *
 * The forward pass and the reverse-mode adjoint (vector-Jacobian product) of
 * the three custom layers of the gradient-Halide chapter, "Custom Neural
 * Network Layers":
 *   stn_*    spatial transformer: affine_grid + bilinear grid_sample
 *   warp_*   FlowNet 2.0 per-pixel warp
 *   bslice_* HDRNet bilateral slice-apply
 * plus, from the §8(f) NEXT rows, the 2-D convolution layer of the paper's
 * scatter-to-gather example (conv_*).
 * Each *_bwd takes "a buffer representing the adjoints" of the layer output
 * and returns the adjoints of the inputs, i.e. df(x, dy) of
 * PAPER.md:2239-2241.  The exact definitions (the paper prints none; its
 * listings are missing) are DESIGN.md R1-R9.
 *
 * Conventions shared by every entry point
 *   Tensors   fp32, C-contiguous (NCHW), no aliasing between inputs and outputs.
 *   Pointers  device pointers (cudaMalloc / torch CUDA tensors) OR host pointers
 *             (pinned or pageable).  All-device calls run entirely on `stream`.
 *             If any pointer is host memory the batch is processed in up to 32
 *             sample chunks on three library-internal streams that are ordered after
 *             `stream` (event wait) and before its later work (event wait back):
 *             per chunk, host inputs are copied H2D into stream-ordered
 *             temporaries (cudaMallocAsync), the kernels run, host outputs are
 *             copied D2H, so copies and kernels of different chunks overlap.
 *             Host outputs are valid once `stream` has been synchronised (pinned
 *             memory: fully asynchronous; pageable: copies may block the caller).
 *   Outputs   always OVERWRITTEN, never accumulated.  A NULL gradient pointer
 *             skips that gradient's work.
 *   Ownership the caller owns every buffer; the library allocates nothing that
 *             outlives a call.  Its only state: the thread-local error string and,
 *             per (thread, device), the internal streams/events of the host-pointer
 *             path and of stn_bwd's side stream (created on first use, reused,
 *             released with the CUDA context).
 *   Workspace *_bwd take an optional device workspace of
 *             rsgrad_bwd_workspace_bytes(...) bytes (same opts: deterministic=1
 *             adds the fixed-point accumulators; stn_bwd always holds one channel
 *             plane's, for AUTO's exact scatter of high fan-in fallback samples).  NULL /
 *             ws_bytes too small (e.g.
 *             0) => the library takes a stream-ordered temporary of that size from
 *             the stream's device's DEFAULT memory pool (cudaMallocAsync) and frees it
 *             in stream order (cudaFreeAsync): nothing is reserved by the library
 *             after the call; caching is the pool's (the caller's) release policy.
 *             (Reading of SURVEY 8(b) "ws_bytes=0 => workspace-free algorithm":
 *             every backward here needs scratch for its fixed-order partial sums,
 *             which is what makes it deterministic, so the free-standing variant is
 *             a stream-ordered temporary rather than a different algorithm;
 *             DESIGN.md "Boundary".)
 *   Devices   every entry point runs on the device of `stream` (made current for
 *             the call, the previous device restored); NULL stream = the current
 *             device.  All pointers must belong to that device (or be host memory).
 *   Errors    no exceptions cross the ABI: a negative rs_status is returned and
 *             rsgrad_last_error() describes it.  Status reflects argument
 *             validation and launch errors (cudaGetLastError) only; kernel
 *             faults surface on the next synchronisation of `stream`.
 *   Threads   re-entrant; concurrent calls on different streams are safe.
 *   Graphs    with device pointers every entry point is stream-capture safe (only
 *             kernel launches, memsets and stream-ordered alloc/free on `stream`;
 *             stn_bwd on a small batch also forks its d_theta kernel onto a library
 *             side stream with an event recorded on `stream` and joins it back with
 *             an event wait before its last kernel -- ordered like `stream`, and part
 *             of a capture of `stream`):
 *             capture it into a CUDA graph and replay it (the per-kernel launch
 *             gaps of a multi-kernel call shrink; bench.py paper_shapes *_graph).
 *             While `stream` is capturing, its device must be the current one.
 *             The host-pointer path is not capturable.
 *   Determinism: with deterministic=1 every result is bitwise reproducible, for
 *             every sample: gathers and fixed-order partial sums as always, and where
 *             a scatter cannot be converted (STN samples with a singular map or a huge
 *             preimage, STN border padding, warp d_input, bicubic fallback samples,
 *             bslice d_grid on grids finer than 8 px per cell) the fixed-point
 *             integer scatter: each term w*g rounded once to a 64-bit
 *             integer at a per-sample scale 2^S (S from max|dy|), summed with integer
 *             atomics (order-free), converted once (absolute error <= n 2^-(S+1) for
 *             n terms, n*max|dy|*P*2^-62), also for the stn3d / Lanczos adjoints.
 *             SCATTER_ATOMIC / SCATTER_PRIV with deterministic=1 => RS_ERR_FLAG.
 */
#ifndef RSGRAD_H
#define RSGRAD_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same object as cudaStream_t / CUstream; NULL = the legacy default stream. */
typedef struct CUstream_st *rs_stream_t;

typedef enum {
    RS_OK = 0,
    RS_ERR_NULL = -1,      /* a required pointer is NULL                      */
    RS_ERR_SHAPE = -2,     /* a dimension is non-positive / degenerate         */
    RS_ERR_ALIGN = -3,     /* reserved (misalignment takes a scalar path)      */
    RS_ERR_FLAG = -4,      /* bad option, or algo not valid for these inputs   */
    RS_ERR_CUDA = -5,      /* CUDA runtime error (message in last_error)       */
    RS_ERR_WORKSPACE = -6  /* workspace could not be obtained                  */
} rs_status;

typedef enum { RS_PAD_ZEROS = 0, RS_PAD_BORDER = 1 } rs_padding;

/* Backward algorithm for the scattered adjoint (convert scatters
 * to gathers where a bounded inverse exists, else "a general scattering operation"
 * with atomics).  What each layer accepts:
 *   stn_bwd  d_input  AUTO, GATHER: cell-owner gather over the affine preimage
 *                     (zeros padding; per-sample fallback to atomics -- or, with
 *                     deterministic=1, the fixed-point scatter -- for singular
 *                     theta / huge preimages); SCATTER_ATOMIC: per-tap global atomics;
 *                     SCATTER_PRIV: per output tile, taps accumulate in a shared-
 *                     memory copy of the tile's input footprint, flushed with one
 *                     global atomic per touched element.  Border padding never
 *                     gathers (no bounded inverse).
 *   warp_bwd d_input  AUTO: row strips -- each lane walks rows of one column and keeps
 *                     its current cell's 4 tap sums in registers (carried down a
 *                     row, merged with the neighbour lane's shared taps and across
 *                     runs of lanes on one cell) before fp32 global atomics; a
 *                     sample where one pre-summed emission covers >= 32 taps (a
 *                     collapsing flow) is then recomputed by the fixed-point
 *                     scatter (needs the workspace rsgrad_ws_bytes reports);
 *                     deterministic=1: the fixed-point scatter;
 *                     SCATTER_ATOMIC: one fp32 atomic per tap (the unconverted
 *                     scatter); SCATTER_PRIV as for STN; GATHER -> RS_ERR_FLAG (an
 *                     arbitrary flow has no bounded inverse).
 *   bslice_bwd d_grid AUTO, SCATTER_PRIV: dual-cell register-privatised
 *                     accumulation + fixed-order partial gather (deterministic;
 *                     cells >= 8 px; finer grids: global atomics, or with
 *                     deterministic=1 the fixed-point scatter); GATHER (D <= 16):
 *                     the pure gather -- every grid node walks the pixels of its
 *                     2 x 2 dual cells (deterministic; each pixel visited 4 times);
 *                     SCATTER_ATOMIC: global atomics.
 * d_theta, d_flow, d_guide and bslice d_input are always gathers. */
typedef enum {
    RS_ALGO_AUTO = 0,
    RS_ALGO_GATHER = 1,
    RS_ALGO_SCATTER_PRIV = 2,
    RS_ALGO_SCATTER_ATOMIC = 3
} rs_algo;

typedef struct {
    int align_corners; /* STN only: 1 (default, R2) or 0          */
    int padding;       /* rs_padding: STN and warp; bslice always clamps     */
    int algo;          /* rs_algo                                            */
    int deterministic; /* 1 => bitwise reproducible results                  */
} rs_opts;

/* NULL opts pointer => {align_corners=1, padding=ZEROS, algo=AUTO, deterministic=0}. */

/* ---------------------------------------------------------------------------
 * Spatial transformer.
 *   x      N x C x H x W        input feature map
 *   theta  N x 2 x 3            per-sample affine, normalised coordinates
 *   y      N x C x Ho x Wo      output
 *   y[n,c,i,j] = bilinear(x[n,c], ix, iy) with (ix, iy) the un-normalised image
 *   of theta_n [xt_j, yt_i, 1]^T (R1); taps outside the image read 0
 *   (zeros) or the coordinate is clamped to the image (border).
 * Shapes: N, C, H, W, Ho, Wo >= 1; align_corners=1 requires Ho, Wo >= 2.
 * ------------------------------------------------------------------------- */
rs_status stn_fwd(const float *x, const float *theta, int N, int C, int H, int W, int Ho,
                  int Wo, const rs_opts *opts, float *y, rs_stream_t stream);

/*   dy      N x C x Ho x Wo     adjoint of y
 *   dx      N x C x H x W       adjoint of x (nullable)
 *   dtheta  N x 2 x 3           adjoint of theta (nullable)
 * GATHER is invalid with border padding (the clamp has no bounded inverse);
 * border padding with deterministic=1 takes the fixed-point scatter for d_input. */
rs_status stn_bwd(const float *x, const float *theta, const float *dy, int N, int C, int H,
                  int W, int Ho, int Wo, const rs_opts *opts, float *dx, float *dtheta,
                  void *workspace, size_t ws_bytes, rs_stream_t stream);

/* ---------------------------------------------------------------------------
 * FlowNet 2.0 warp: y[n,c,y,x] = bilinear(x[n,c], x+u, y+v),
 * flow N x 2 x H x W in pixels, channel 0 = u (horizontal).  DESIGN.md R4.
 * ------------------------------------------------------------------------- */
rs_status warp_fwd(const float *x, const float *flow, int N, int C, int H, int W,
                   const rs_opts *opts, float *y, rs_stream_t stream);

/*   dx N x C x H x W (nullable), dflow N x 2 x H x W (nullable).
 * GATHER is invalid (arbitrary flow has no bounded inverse). */
rs_status warp_bwd(const float *x, const float *flow, const float *dy, int N, int C, int H,
                   int W, const rs_opts *opts, float *dx, float *dflow, void *workspace,
                   size_t ws_bytes, rs_stream_t stream);

/* ---------------------------------------------------------------------------
 * HDRNet bilateral slice-apply.
 *   grid   N x 12 x D x Gh x Gw   affine coefficients, q = 4*o + i (3x4 row-major)
 *   guide  N x H x W              guidance map (any real value; clamped planes)
 *   x      N x 3 x H x W          input image
 *   y      N x 3 x H x W          y_o = sum_i A_{4o+i} x_i + A_{4o+3},
 *   A = trilinear tent slice of grid at ((x+.5)Gw/W-.5, (y+.5)Gh/H-.5, guide*D-.5)
 *   with indices clamped to the grid (R5-R7).  opts.padding ignored.
 * ------------------------------------------------------------------------- */
rs_status bslice_fwd(const float *grid, const float *guide, const float *x, int N, int H,
                     int W, int D, int Gh, int Gw, const rs_opts *opts, float *y,
                     rs_stream_t stream);

/*   dgrid N x 12 x D x Gh x Gw, dguide N x H x W, dx N x 3 x H x W (each nullable). */
rs_status bslice_bwd(const float *grid, const float *guide, const float *x, const float *dy,
                     int N, int H, int W, int D, int Gh, int Gw, const rs_opts *opts,
                     float *dgrid, float *dguide, float *dx, void *workspace, size_t ws_bytes,
                     rs_stream_t stream);

/* ---------------------------------------------------------------------------
 * 2-D convolution layer: the scatter-vs-gather example of
 * PAPER.md:703-733, "output(x) = input(x - r.x) * kernel(r.x)" in 2-D with
 * channels, centred (R10):
 *   y[n,co,y,x] = sum_{ci<Ci,ry<kh,rx<kw} x[n,ci, y-ry+kh/2, x-rx+kw/2] * k[co,ci,ry,rx]
 *   x N x Ci x H x W, k Co x Ci x kh x kw, y N x Co x H x W, zero outside the image.
 * DEVICE pointers only (k and dk are shared by the whole batch); 1 <= kh, kw <= 7
 * and Ci small enough for the d_kernel tile to fit in shared memory,
 * 4 * (Ci*(15+kh)*(32+kw) + 2048*ceil(Co/4)) <= 200 KB (Ci <= 68 at 3x3 with Co = 16),
 * else RS_ERR_SHAPE.  opts.padding/align_corners ignored.
 * ------------------------------------------------------------------------- */
rs_status conv_fwd(const float *x, const float *k, int N, int Ci, int Co, int H, int W, int kh,
                   int kw, const rs_opts *opts, float *y, rs_stream_t stream);

/*   dx N x Ci x H x W (nullable): AUTO/GATHER = the converted, sheared gather
 *   "d_input(x) += d_output(x + r.x) * kernel(r.x)" over zero-padded d_output
 *   (PAPER.md:721-724), deterministic; SCATTER_ATOMIC = the unconverted scatter
 *   "d_input(ro.y - ro.x) += d_output(ro.y) * kernel(ro.x)" with atomics
 *   (memset + red.global.add, not deterministic).
 *   SCATTER_PRIV is refused (RS_ERR_FLAG).
 *   dk Co x Ci x kh x kw (nullable): sum over the batch and pixels of dy x shifted x,
 *   per-block partials in the workspace + a fixed-order sum (deterministic). */
rs_status conv_bwd(const float *x, const float *k, const float *dy, int N, int Ci, int Co, int H,
                   int W, int kh, int kw, const rs_opts *opts, float *dx, float *dk,
                   void *workspace, size_t ws_bytes, rs_stream_t stream);

/* ---------------------------------------------------------------------------
 * Checkpointing study: the gradient of
 *   loss = sum (conv(in, k) - target)^2,  conv = the conv_* layer with Ci = Co = 1,
 *   d_in(u) = sum_r k(r) R(u + r - p),  R = 2 (conv(in) - target), zero outside,
 * "a cross correlation of 2*(convolved-target) with kernel".
 *   in, target, d_in  N x H x W (device);  k  kh x kw, HOST pointer (copied into the
 *   kernel parameters; 1 <= kh, kw <= 7).
 *   schedule  RS_SCHED_ROOT   R written to the workspace, then gathered (compute_root)
 *             RS_SCHED_INLINE R recomputed at every tap (compute_inline)
 *             RS_SCHED_AT     R per 32 x 32 tile of d_in in shared memory (compute_at)
 * The paper's 2560 x 1600 image with 1 x 5 and 3 x 5 kernels.
 * ------------------------------------------------------------------------- */
typedef enum { RS_SCHED_ROOT = 0, RS_SCHED_INLINE = 1, RS_SCHED_AT = 2 } rs_schedule;
rs_status convloss_grad(const float *in, const float *k, const float *target, int N, int H, int W,
                        int kh, int kw, rs_schedule schedule, float *d_in, void *workspace,
                        size_t ws_bytes, rs_stream_t stream);

/* Upsampling by 4, output(x, y) = input(x/4, y/4):
 *   x N x C x H x W -> y N x C x 4H x 4W;  the adjoint is the converted gather
 *   d_input(x) = sum_{r < 4 x 4} d_output(4x + r), deterministic.
 * Device pointers only. */
rs_status upsample4_fwd(const float *x, int N, int C, int H, int W, float *y, rs_stream_t stream);
rs_status upsample4_bwd(const float *dy, int N, int C, int H, int W, float *dx, rs_stream_t stream);

/* ---------------------------------------------------------------------------
 * STN variants ("changing the interpolation scheme
 * ... or interpolating over more dimensions").  Device pointers only; zeros padding
 * only (opts.padding = RS_PAD_BORDER => RS_ERR_FLAG); opts.align_corners as stn_*.
 * d_theta is a fixed-order fp64 sum of per-block partials.  d_input:
 *   stn_bicubic_bwd  GATHER or deterministic=1: the converted gather -- each input pixel
 *                    enumerates the affine preimage of (x-2, x+2) x (y-2, y+2) with exact
 *                    fp64 membership (a singular map or a window > 1024 output pixels
 *                    falls back to reds for that sample, to the fixed-point scatter
 *                    with deterministic=1); AUTO / SCATTER_ATOMIC: memset +
 *                    red.global.add per tap in the d_theta pass (measured faster).
 *   stn3d_bwd        the atomic scatter (GATHER => RS_ERR_FLAG); deterministic=1: the
 *                    fixed-point scatter (bitwise reproducible).
 * SCATTER_PRIV => RS_ERR_FLAG.
 *   stn_bicubic_*  theta N x 2 x 3, x N x C x H x W, y N x C x Ho x Wo: Keys' cubic
 *                  convolution (A = -0.75) over the 4 x 4 taps floor(i)-1 .. floor(i)+2
 *                  (= torch grid_sample mode='bicubic', zeros; R12).
 *   stn3d_*        theta N x 3 x 4, x N x C x D x H x W, y N x C x Do x Ho x Wo:
 *                  5-D affine_grid + trilinear grid_sample (zeros).
 * ------------------------------------------------------------------------- */
rs_status stn_bicubic_fwd(const float *x, const float *theta, int N, int C, int H, int W, int Ho,
                          int Wo, const rs_opts *opts, float *y, rs_stream_t stream);
rs_status stn_bicubic_bwd(const float *x, const float *theta, const float *dy, int N, int C, int H,
                          int W, int Ho, int Wo, const rs_opts *opts, float *dx, float *dtheta,
                          void *workspace, size_t ws_bytes, rs_stream_t stream);
/*   stn_lanczos_*  as stn_bicubic_* with 6 x 6 taps floor(i)-2 .. floor(i)+3 and the
 *                  Lanczos-3 kernel L(x) = sinc(x) sinc(x/3), |x| < 3 (R13);
 *                  d_input by the atomic scatter (GATHER => RS_ERR_FLAG), with
 *                  deterministic=1 the fixed-point scatter; workspace layer 7. */
rs_status stn_lanczos_fwd(const float *x, const float *theta, int N, int C, int H, int W, int Ho,
                          int Wo, const rs_opts *opts, float *y, rs_stream_t stream);
rs_status stn_lanczos_bwd(const float *x, const float *theta, const float *dy, int N, int C, int H,
                          int W, int Ho, int Wo, const rs_opts *opts, float *dx, float *dtheta,
                          void *workspace, size_t ws_bytes, rs_stream_t stream);
rs_status stn3d_fwd(const float *x, const float *theta, int N, int C, int D, int H, int W, int Do,
                    int Ho, int Wo, const rs_opts *opts, float *y, rs_stream_t stream);
rs_status stn3d_bwd(const float *x, const float *theta, const float *dy, int N, int C, int D, int H,
                    int W, int Do, int Ho, int Wo, const rs_opts *opts, float *dx, float *dtheta,
                    void *workspace, size_t ws_bytes, rs_stream_t stream);

/* Workspace (bytes) *_bwd wants for these shapes.  layer: 0 = STN (uses
 * N,C,H,W,Ho,Wo), 1 = warp (N,C,H,W), 2 = bslice (N,H,W,D,Gh,Gw), 3 = conv
 * (N, C = Ci, H, W, D = Co, Gh = kh, Gw = kw), 4 = convloss_grad (N, H, W: the
 * RS_SCHED_ROOT residual), 5 = stn_bicubic (N, Ho, Wo: d_theta partials, coordinate
 * tables, N fallback flags), 6 = stn3d (N, Ho, Wo, D = Do; with deterministic=1 also C, H, W
 * and Gh = depth of the input volume), 7 = stn_lanczos (N, Ho, Wo; deterministic=1: C, H, W);
 * unused arguments are ignored.
 * opts->deterministic = 1 adds the fixed-point accumulators of one sample
 * (8 * C * H * W bytes) for layers 0, 1, 5, 6 and 7; layer 0 (stn) always includes one
 * channel plane (8 * H * W bytes: AUTO's exact scatter of high fan-in fallback samples).
 * Returns 0 for an unknown layer. */
size_t rsgrad_bwd_workspace_bytes(int layer, int N, int C, int H, int W, int Ho, int Wo, int D,
                                  int Gh, int Gw, const rs_opts *opts);

/* Thread-local description of the last error on this thread ("" if none). */
const char *rsgrad_last_error(void);

/* Library version string, e.g. "rsgrad 0.1.0 sm_100a". */
const char *rsgrad_version(void);

/* Caller-owned device staging buffer for the host-pointer path on the calling thread
 * and the current device: when it holds 3 streams x (the host tensors of one sample
 * chunk + that chunk's workspace), calls carve their staging from it instead of taking
 * stream-ordered temporaries per call.  Calls that use it are serialised on an event
 * (each waits until the previous user is done).  buf = NULL unregisters (waiting until
 * the last user is done).  The caller keeps ownership and must not free `buf` while
 * registered.  RS_ERR_FLAG if buf is not device memory. */
rs_status rsgrad_set_host_staging(void *buf, size_t bytes);

/* Number of kernels the library enqueued on this thread since the last reset
 * (launch accounting for bench.py's gpu_launches). */
unsigned long long rsgrad_launch_count(int reset);

#ifdef __cplusplus
}
#endif

#endif /* RSGRAD_H */
