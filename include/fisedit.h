/*
 * fisedit.h — C ABI of the B200 sparse-edit kernels (libfisedit.so).
 *
 * Plain C: device pointers, sizes, a cudaStream_t passed as void*, int status.
 * No torch types. Caller owns every buffer (activations, caches, workspaces);
 * no entry point allocates, synchronises the device or reads device memory on
 * the host. All entry points are reentrant per stream and graph-capturable.
 *
 * Each entry point replaces a reference (sparsedit 0.1.0) interface — see the
 * per-function comment for the file:line it stands in for.
 *
 * Step indexing: every fis_ref may carry a step_stride. The kernels read the
 * current step t from *step (device int, NULL => 0) and address
 * ptr + t*step_stride. This lets one captured CUDA graph replay every denoising
 * step of an edit (the per-step cache slabs differ only by t*stride).
 */
#ifndef FISEDIT_H
#define FISEDIT_H

#ifdef __cplusplus
extern "C" {
#endif

#define FIS_ABI_VERSION 1

/* status codes (mapped to sparsedit exceptions by the Python wrapper) */
#define FIS_OK 0
#define FIS_ERR_SHAPE 1        /* ContractViolation */
#define FIS_ERR_CACHE_MISS 2   /* CacheMissError */
#define FIS_ERR_UNSUPPORTED 3  /* ContractViolation (unsupported combination) */
#define FIS_ERR_LAUNCH 4       /* RuntimeError (CUDA launch failure) */

/* element types */
#define FIS_F32 0
#define FIS_BF16 1

typedef struct {
    void* ptr;              /* base address (device) */
    long long step_stride;  /* bytes added per step index */
    int ld;                 /* elements between consecutive rows / pixels */
    int dtype;              /* FIS_F32 | FIS_BF16 */
} fis_ref;

/* A selectable feature map (select-on-read):
 *   value(q, c) = index ? (index[q] >= 0 ? fresh[index[q]*ld + c] : cache[q*ld + c])
 *                       : fresh[q*ld + c]
 * for source pixel q = sy*w + sx. */
typedef struct {
    fis_ref fresh;
    fis_ref cache;
    const int* index;       /* [h*w] pixel -> fresh row, -1 = not fresh; NULL => fresh is a full map */
    int h, w;               /* source pixel grid */
    int c;                  /* channels contributed by this source */
    int up;                 /* 1: consumer pixel (y,x) reads source pixel (y>>1, x>>1) (nearest upsample) */
} fis_src;

#define FIS_A_ROWS 0    /* A[r,k] = a[(rows ? rows[r] : r)*ld + k] */
#define FIS_A_CONV3X3 1 /* implicit 3x3 same-padding conv over concat(src[0], src[1]), K = 9*Cin, tap-major */

#define FIS_EPI_NONE 0
#define FIS_EPI_GN_SILU 1  /* y = gamma*(v-mean_g)/sqrt(var_g+eps)+beta ; out = silu(y) */
#define FIS_EPI_STEP 2     /* out = lat - step_scale * v   (unet.py:693,883) */

/* Gather-GEMM:  D[r, n] = epilogue( sum_k A[r,k] * B[n,k] )   (B is [N, K], K contiguous)
 * Replaces: conv2d / _conv_accumulate (tensors.py:76-126), sparse_conv gather+conv+scatter
 * (sparse.py:143-223), _project (sparse.py:261-262), attention_scores/apply_attention
 * GEMMs (tensors.py:183-200), _text_kv (unet.py:476-479). */
typedef struct {
    int m, n, k;
    int a_mode;
    fis_ref a;
    const int* rows;        /* output pixel (CONV) / A row (ROWS) of GEMM row r; NULL => r */
    int out_h, out_w;       /* CONV: output pixel grid */
    int nsrc;
    fis_src src[2];
    fis_ref b;
    /* epilogue, applied in this order */
    float alpha;            /* v = acc*alpha */
    const float* bias;      /* v += bias[n] */
    fis_ref bias2;          /* v += bias2[n] (separately rounded; e.g. time bias row of step t) */
    fis_ref pre;            /* optional store of v (raw layer output, for recording) */
    int epi;
    fis_ref gn_mean, gn_var;/* [groups] f32 */
    const float* gamma;
    const float* beta;
    int groups;
    float eps;
    fis_ref pre2;           /* GN_SILU: optional store of y before SiLU (norm output) */
    fis_ref lat;            /* STEP: latent rows (may alias d) */
    float step_scale;
    fis_ref res;            /* v += res[r, n] (residual) */
    fis_ref d;              /* output */
    int d_trans;            /* 1: store D[n*ld + r] */
    int n_split;            /* >0: columns n >= n_split go to d2 at column n - n_split (fused QKV) */
    fis_ref d2;
    int d2_trans;
    const int* d_rows;      /* optional row remap for the output (and res/lat/pre): row = d_rows[r];
                               d_rows[r] < 0: row r is computed but not stored */
    /* scheduling */
    int splits;             /* split-K factor; 0 = choose from the tile shape and SM count */
    float* ws;              /* splits*m*n floats when splits > 1 */
    long long ws_floats;    /* capacity of ws (bounds the automatic split choice) */
    int* counters;          /* per-tile arrival counters (zeroed, self-resetting) */
    const int* step;
    int impl;               /* 0 auto, 1 SIMT fp32-accumulate, 2 tcgen05 bf16, 3 tcgen05 3xTF32 on fp32
                               operands (SIMT when the shape is not supported) */
    int static_meta;        /* 1: rows/index lists are not written by the preceding kernel, so the
                               gather metadata may be read before the programmatic-launch wait */
    int m_halo;             /* CONV with rows + d_rows: 1 = the GEMM rows are runs of horizontally
                               adjacent pixels, each run framed by its left / right neighbour pixel
                               (or -1 at the image border) as rows with d_rows = -1 (not stored); the
                               persistent kernel then stages each channel block once per kernel row
                               (dy) and reads the three dx taps as 1-row shifts (fis_gemm_halo.cu) */
} fis_gemm_args;

int fis_gemm(const fis_gemm_args* args, void* stream);
/* which kernel fis_gemm picks for these arguments: 0 SIMT, 1 per-op tcgen05 (split-K clusters),
 * 2 persistent large-M tcgen05 (TMA / gather4 staging), 3 per-op tcgen05 3xTF32, 4 halo-staged
 * persistent gather conv (m_halo), 5 few-input-channel 3x3 conv on the FMA pipes (the latent stem
 * conv, C_in <= 8), 6 persistent 2-SM CTA-pair GEMM (tcgen05 cta_group::2, TMA-staged A); host-only */
int fis_gemm_kernel_kind(const fis_gemm_args* a);
/* number of persistent-kernel launches so far (diagnostics / tests) */
long long fis_gemm_big_launch_count(void);
/* number of 2-SM (CTA pair) GEMM launches so far (diagnostics / tests) */
long long fis_gemm_pair_launch_count(void);
/* workspace floats / counters needed for a given problem */
long long fis_gemm_ws_floats(int m, int n, int splits);
int fis_gemm_counters(int m, int n);

/* Group-norm statistics over a full map: mean/var per group in f64, rounded to f32.
 * Replaces group_norm's reduction (tensors.py:129-146). */
typedef struct {
    int hw, c, groups;
    fis_ref x;              /* [n_img * hw, ld] */
    fis_ref mean, var;      /* [n_img][groups] f32 */
    const int* step;
    int n_img;              /* stacked images (batched requests), statistics per image; 0/1 = one */
} fis_gn_stats_args;
int fis_gn_stats(const fis_gn_stats_args* a, void* stream);

/* Row-wise group normalisation with given stats (+ optional SiLU).
 * Replaces normalize_with_group_stats (tensors.py:149-180), sparse_group_norm
 * (sparse.py:226-251) and _silu (unet.py:291-293). */
typedef struct {
    int rows, c, groups;
    float eps;
    fis_ref x; const int* x_rows;
    fis_ref mean, var;
    const float* gamma;
    const float* beta;
    fis_ref y_norm;         /* optional */
    fis_ref y_silu;         /* optional */
    const int* y_rows;
    const int* step;
    int img_rows;           /* > 0: row r uses the statistics of image r / img_rows (mean/var [img][groups]) */
    const int* row_img;     /* optional per-row image index (overrides img_rows) */
} fis_gn_apply_args;
/* Dense group norm computing its own statistics (group_norm, tensors.py:129-146, + SiLU):
 * rows = n_img * img_rows (img_rows = 0: one image), statistics written to mean / var
 * [img][groups]; no row lists. One launch for bf16 maps with 8 | channels per group. */
int fis_gn(const fis_gn_apply_args* a, void* stream);
/* kernel launches one fis_gn call makes: 1 (fused statistics + normalise) or 2 */
int fis_gn_launches(const fis_gn_apply_args* a);
int fis_gn_apply(const fis_gn_apply_args* a, void* stream);

/* Row softmax of scaled scores, optional controlled-mode column substitution.
 * Replaces attention_scores (tensors.py:183-192) and ControlledMode.cross_attn's
 * column pinning + renormalisation (unet.py:555-566). */
typedef struct {
    int rows, cols, pad_cols;
    fis_ref s;              /* f32 scores [rows, ld] */
    float scale;
    fis_ref p;              /* probabilities [rows, ld], columns [cols, pad_cols) zeroed */
    fis_ref map;            /* optional f32 copy [rows, ld] (CROSS_ATTN_MAP recording) */
    fis_ref cached;         /* controlled mode: cached map [rows, ld] (old-prompt columns) */
    int verbatim;           /* 1: p = cached (all tokens shared) */
    int npairs;
    const int* pair_old;
    const int* pair_new;
    const int* step;
} fis_softmax_args;
int fis_softmax(const fis_softmax_args* a, void* stream);

/* Fused tensor-core attention (tcgen05): out = res + softmax(Q K^T * scale) V for one query
 * tile of 128 rows x one output-channel slice per CTA; S and the O slice accumulate in TMEM,
 * P goes through a swizzled shared-memory tile into the P.V MMA. Replaces attention_scores +
 * apply_attention + the residual add for self- and cross-attention (sparse.py:265-361,
 * tensors.py:183-200, unet.py:456-457).  bf16 Q/K/V^T, d % 64 == 0. */
typedef struct {
    int m, n_keys, d, dv;   /* queries, keys, head dim (= reduction dim of Q K^T), value dim */
    fis_ref q;              /* [m, ld] */
    fis_ref k;              /* [n_keys, ld] */
    fis_ref vt;             /* [dv, ld]: V transposed (keys contiguous) */
    float scale;
    fis_ref res;            /* [m, ld] residual (may be NULL) */
    fis_ref pre;            /* optional store of the attention output before the residual */
    fis_ref out;            /* [m, ld] */
    const int* step;
    /* ragged segments (batched requests): queries [q_seg[2s], q_seg[2s+1]) attend to keys
     * [k_seg[2s], k_seg[2s+1]) only; nseg = 0: one segment of m queries x n_keys keys */
    int nseg;
    int max_seg_q;          /* largest q_seg[s+1] - q_seg[s] (sizes the grid) */
    const int* q_seg;       /* [2 * nseg] device (begin, end) pairs */
    const int* k_seg;       /* [2 * nseg] device (begin, end) pairs */
    int max_seg_k;          /* > 0: longest key run; lets the value slices of a query tile share
                               one P (computed once into ws) instead of recomputing S */
    void* ws;               /* P scratch: [m][128 * ceil(max_seg_k / 128)] bf16 (may be NULL) */
    long long ws_bytes;
} fis_attn_args;
int fis_attn(const fis_attn_args* a, void* stream);
/* kernel launches one fis_attn call makes: 1, or 2 when the value slices share P (0: unsupported) */
int fis_attn_launches(const fis_attn_args* a);
/* workspace bytes fis_attn can use for m queries, runs of <= max_keys keys and dv value columns
 * (P sharing scratch, or the split-KV partials of long runs + completion counters); pass it
 * zero-initialised as ws / ws_bytes */
long long fis_attn_ws_bytes(int m, int max_keys, int dv);

/* 2x2 average pool with select-on-read of the finer map (unet.py:296-298).
 * Output rows are coarse pixels rows[i] (NULL => all (h/2)*(w/2)). */
typedef struct {
    int n, c;
    fis_src src;
    const int* rows;
    fis_ref out;
    const int* step;
} fis_pool_args;
int fis_pool2(const fis_pool_args* a, void* stream);
/* Nearest 2x upsample (unet.py:301-302) of the (dense) source map src [img][h][w][c] into
 * out [img][2h][2w][c]; n = output pixels. Materialises the coarse half of a fuse concat so the
 * fuse conv of a dense level can stage its A operand with TMA (stacked requests). */
int fis_up2(const fis_pool_args* a, void* stream);

/* Materialise a full map from a selectable source: out[q] = value(q) for all q.
 * Replaces the cached-copy + pixel scatter of sparse ops (sparse.py:209-220,248-250,298-299). */
typedef struct {
    int c;
    fis_src src;
    fis_ref out;            /* [h*w, ld] */
    const int* step;
} fis_materialize_args;
int fis_materialize(const fis_materialize_args* a, void* stream);

/* Mask detection, one fused CTA: Σ_t channel-mean |X_t - Y_t| (f64), min-max
 * normalise, Otsu over 256 candidates (numpy pairwise-sum order, bit-exact),
 * threshold, square dilation.  Replaces accumulate_diff / otsu_threshold /
 * dilate (masks.py:117-192).  x: t-th latent at x.ptr + (t-1)*x.step_stride,
 * layout [hw, c] f32; same for y.
 * result[0]=epsilon, [1]=objective (f64); flags[0]=no_edit, [1]=degenerate. */
typedef struct {
    int h, w, c, t1, t2, radius;
    fis_ref x, y;
    float* values;          /* [h*w] normalised diff (DiffMap.values) */
    unsigned char* raw_mask;/* [h*w] threshold mask before dilation */
    unsigned char* mask;    /* [h*w] dilated mask */
    double* result;
    int* flags;
    const float* values_in; /* optional: skip the diff phase and threshold these values (otsu_threshold) */
} fis_mask_detect_args;
int fis_mask_detect(const fis_mask_detect_args* a, void* stream);
long long fis_mask_detect_smem(int h, int w);

/* Mask plan, one fused CTA: OR-pool pyramid, per-level row-major active-pixel
 * lists + pixel->row index maps, per-level active 2x2-tile lists (the gather
 * plan origins of sparse.py:91-140 for 3x3 kernels) via warp
 * ballot + block prefix sum.  Replaces build_pyramid (masks.py:195-210),
 * select_gather_plan's origins/cost and np.flatnonzero (sparse.py:289,327). */
#define FIS_MAX_LEVELS 8
typedef struct {
    int h, w, levels;
    int radius;                         /* square dilation of the input mask first (masks.py:180-192) */
    const unsigned char* mask;          /* [h*w] level-0 mask (before dilation) */
    unsigned char* bits[FIS_MAX_LEVELS];/* [h_l*w_l] pyramid levels (may be NULL) */
    int* rows[FIS_MAX_LEVELS];          /* [h_l*w_l] active pixel list, row-major */
    int* index[FIS_MAX_LEVELS];         /* [h_l*w_l] pixel -> row or -1 */
    int* tiles[FIS_MAX_LEVELS];         /* [ceil(h_l/2)*ceil(w_l/2)] active tile ids (ty*tw+tx), may be NULL */
    int* counts;                        /* [2*levels]: active pixels per level, active tiles per level */
} fis_mask_plan_args;
int fis_mask_plan(const fis_mask_plan_args* a, void* stream);

/* profiling: phase timestamps (%globaltimer ns) of CTA (0,0,0) of tcgen05 GEMM launches */
int fis_trace(int on);
int fis_trace_read(unsigned long long* out16);
int fis_trace_read_ctas(unsigned long long* out2048); /* per CTA: entry, MMA done, cluster sync, exit */
/* launch trace: buf (device, >= 16 + 16 * 4096 u64, zeroed) receives, per kernel launch in start
   order, CTA (0,0,0)'s %globaltimer phase stamps (buf[0] = launch counter); NULL switches it off */
int fis_trace_launches(unsigned long long* buf);

/* misc */
int fis_abi_version(void);
const char* fis_last_error(void);
int fis_device_sm_count(void);

#ifdef __cplusplus
}
#endif
#endif /* FISEDIT_H */
