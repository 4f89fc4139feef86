// Halo-staged persistent gather-conv (tcgen05, sm_100a) for the stacked sparse convs.
//
// The gathered 3x3 convs of the stacked step were bound by staging A: every 64-channel K block of
// every tap fetched its 128 scattered rows again (9 fetches of each source row per channel block).
// Here the GEMM rows are runs of horizontally adjacent active pixels, each run framed by its left /
// right neighbour pixel (rows whose output is not stored, d_rows = -1; fis_gemm_args.m_halo). For a
// tile of 128 rows and one channel block, the producers stage 130 rows [m0-1, m0+129) of the source
// shifted by one kernel row dy (3 stagings per channel block instead of 9), in the no-swizzle
// K-major UMMA layout with the 8 16-byte K chunks as planes: row s of plane j at j*PLANE + 16*s.
// Tap (dy, dx) of row r is staging row r + 1 + dx, so its A operand is the same staging buffer with
// the descriptor start moved by (1 + dx) * 16 bytes (LBO = PLANE, SBO = 128 B): no copies.
//
//   warps 0-3 : A producers (cp.async, select-on-read of the fresh compact rows / the cached slab,
//               nearest upsample of the coarse concat half, zero rows outside the image)
//   warp 4    : B producer (TMA {64 x 160} boxes of the tap-major weights, 128B swizzle)
//   warp 5    : TMEM allocator + MMA issuer (tcgen05.mma.cta_group::1.kind::f16, M=128)
//   warps 6-9 : epilogue (TMEM -> bias -> bf16 rows d_rows[r], skipping framing rows)
// Tiles are persistent over CTAs, N-fastest (consecutive CTAs share the staged A in L2).
#include "fis_tc.cuh"
#include "fis_tma.cuh"
#include <cstring>

const CUtensorMap* fis_weight_map(const void* base, long long n, long long k, long long ld, int box);

namespace fis {
namespace halo {

using namespace fis::tc;

constexpr int THREADS = 320, A_WARPS = 4, B_WARP = 4, MMA_WARP = 5, EPI_WARP0 = 6;
constexpr int SROWS = BM + 2;                  // staged rows: the tile plus one framing row each side
constexpr int PLANE = SROWS * 16;              // bytes per 16-byte K chunk plane
constexpr int A_SLOT = 8 * PLANE;              // one (channel block, dy) staging: 16,640 B
constexpr int NA = 3, NB = 3;

struct Layout {
    int bn, bstage, total;
};
__host__ __device__ inline Layout layout(int bn) {
    Layout l;
    l.bn = bn;
    l.bstage = bn * 128;
    // A slots + B stages + barriers + source table [3][SROWS][2] + bias table + align
    l.total = NA * A_SLOT + NB * l.bstage + 512 + 3 * SROWS * 2 * 4 + 2 * bn * 4 + 1024;
    return l;
}

FIS_DEV uint64_t none_desc(uint32_t saddr) {
    // K-major, no swizzle: ((8, m), 2) core matrices, SBO = 128 B between 8-row groups, LBO = PLANE
    // between the two 16-byte K chunks of one MMA (version 1, layout type 0)
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((PLANE >> 4) & 0x3FFF) << 16) |
           ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
}
FIS_DEV void tma2d(uint32_t dst, const void* tmap, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
FIS_DEV void arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
FIS_DEV void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
FIS_DEV void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// select-on-read source of staged row s (GEMM row m0 - 1 + s) shifted by dy, segment seg:
// >= 0 fresh row (or full-map pixel), <= -2 cache pixel (-2 - q), SEL_ZERO zero row
FIS_DEV int halo_src(const fis_gemm_args& a, int i, int dy, int seg) {
    if (i < 0 || i >= a.m) return SEL_ZERO;
    const int p = __ldg(a.rows + i);
    if (p < 0) return SEL_ZERO;
    const fis_src& s = a.src[seg];
    const int ipx = a.out_h * a.out_w;
    const int img = p / ipx, lp = p - img * ipx;
    const int y = lp / a.out_w + dy, x = lp - (lp / a.out_w) * a.out_w;
    if (y < 0 || y >= a.out_h) return SEL_ZERO;
    const int q = img * s.h * s.w + (s.up ? (y >> 1) * s.w + (x >> 1) : y * s.w + x);
    if (!s.index) return q;
    const int f = __ldg(s.index + q);
    return f >= 0 ? f : -2 - q;
}

__global__ void __launch_bounds__(THREADS, 1)
    gemm_halo_kernel(const fis_gemm_args a, const __grid_constant__ CUtensorMap tmap_b, int bn) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const Layout L = layout(bn);
    unsigned char* bbuf = smem + NA * A_SLOT;
    uint64_t* a_full = (uint64_t*)(bbuf + NB * L.bstage);
    uint64_t* a_empty = a_full + NA;
    uint64_t* b_full = a_empty + NA;
    uint64_t* b_empty = b_full + NB;
    uint64_t* acc_full = b_empty + NB;   // [2]
    uint64_t* acc_empty = acc_full + 2;  // [2]
    uint32_t* tmem_slot = (uint32_t*)(acc_empty + 2);
    int* srctab = (int*)(smem + NA * A_SLOT + NB * L.bstage + 512);  // [3][SROWS][2]
    float* biastab = (float*)(srctab + 3 * SROWS * 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tiles_n = (a.n + bn - 1) / bn, tiles_m = (a.m + BM - 1) / BM, ntiles = tiles_m * tiles_n;
    const int cin0 = a.src[0].c, cin = cin0 + (a.nsrc > 1 ? a.src[1].c : 0);
    const int ncb = cin / 64;
    const int nsub = bn > 256 ? 2 : 1, bns = bn / nsub;
    // two TMEM accumulators when they fit: tile i's epilogue overlaps tile i+1's main loop
    const int nbuf = 2 * bn <= 512 ? 2 : 1;

    if (tid == 0) {
        for (int i = 0; i < NA; i++) {
            mbar_init(a_full + i, A_WARPS * 32);
            mbar_init(a_empty + i, 1);
        }
        for (int i = 0; i < NB; i++) {
            mbar_init(b_full + i, 1);
            mbar_init(b_empty + i, 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(acc_full + b, 1);
            mbar_init(acc_empty + b, 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == B_WARP && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_b) : "memory");
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int t = cur_step(a.step);
    pdl_trigger();
    pdl_wait();

    if (warp < A_WARPS) {
        // ------------------------------------------------------------ A producers
        const char* f0 = a.src[0].fresh.ptr ? ref_base(a.src[0].fresh, t) : nullptr;
        const char* f1 = a.nsrc > 1 && a.src[1].fresh.ptr ? ref_base(a.src[1].fresh, t) : nullptr;
        const char* k0 = a.src[0].cache.ptr ? ref_base(a.src[0].cache, t) : nullptr;
        const char* k1 = a.nsrc > 1 && a.src[1].cache.ptr ? ref_base(a.src[1].cache, t) : nullptr;
        const long long lf0 = a.src[0].fresh.ld * 2ll, lf1 = a.src[1].fresh.ld * 2ll;
        const long long lc0 = a.src[0].cache.ld * 2ll, lc1 = a.src[1].cache.ld * 2ll;
        const char* dummy = (const char*)a.b.ptr;
        const uint32_t abase = smem_u32(smem);
        int it = 0, last_m = -1;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int mt = tile / tiles_n;
            if (mt != last_m) {  // source table of the tile's staged rows (all dy, both segments)
                named_sync(2, A_WARPS * 32);  // every producer is done issuing loads from the old table
                last_m = mt;
                for (int e = tid; e < 3 * SROWS * a.nsrc; e += A_WARPS * 32) {
                    const int seg = e % a.nsrc, s = (e / a.nsrc) % SROWS, dyi = e / (a.nsrc * SROWS);
                    srctab[(dyi * SROWS + s) * 2 + seg] = halo_src(a, mt * BM - 1 + s, dyi - 1, seg);
                }
                named_sync(2, A_WARPS * 32);
            }
            for (int cb = 0; cb < ncb; cb++) {
                const int seg = cb * 64 >= cin0 ? 1 : 0;
                const int c = cb * 64 - (seg ? cin0 : 0);
                for (int dyi = 0; dyi < 3; dyi++, it++) {
                    const int slot = it % NA;
                    if (it >= NA) mbar_wait(a_empty + slot, ((it / NA) & 1) ^ 1);
                    const uint32_t sbase = abase + slot * A_SLOT;
                    const int* st = srctab + dyi * SROWS * 2 + seg;
                    const char* fb = seg ? f1 : f0;
                    const char* kb = seg ? k1 : k0;
                    const long long lf = seg ? lf1 : lf0, lc = seg ? lc1 : lc0;
                    for (int e = tid; e < SROWS * 8; e += A_WARPS * 32) {
                        const int s = e >> 3, j = e & 7;
                        const int v = st[s * 2];
                        const char* src = v == SEL_ZERO ? nullptr
                                          : v >= 0      ? fb + (long long)v * lf + (c + j * 8) * 2
                                                        : kb + (long long)(-2 - v) * lc + (c + j * 8) * 2;
                        cp_async16(sbase + j * PLANE + s * 16, src ? (const void*)src : (const void*)dummy, src != nullptr);
                    }
                    cp_async_arrive_noinc(a_full + slot);
                }
            }
        }
    } else if (warp == B_WARP) {
        // ------------------------------------------------------------ B producer (TMA)
        if (lane == 0) {
            const uint32_t bb = smem_u32(bbuf);
            int it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int n0 = (tile % tiles_n) * bn;
                for (int cb = 0; cb < ncb; cb++)
                    for (int tap = 0; tap < 9; tap++, it++) {
                        // K order of the loop: channel block, then kernel row dy, then dx (tap = 3 dy + dx)
                        const int s = it % NB;
                        if (it >= NB) mbar_wait(b_empty + s, ((it / NB) & 1) ^ 1);
                        arrive_expect_tx(b_full + s, (uint32_t)(bn * 128));
                        for (int j = 0; j < nsub; j++)
                            tma2d(bb + s * L.bstage + j * bns * 128, &tmap_b, tap * cin + cb * 64, n0 + j * bns, b_full + s);
                    }
            }
        }
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(bns >> 3) << 17) |
                               ((uint32_t)(BM >> 4) << 24);
        const uint32_t abase = smem_u32(smem), bb = smem_u32(bbuf);
        int ia = 0, ib = 0, lt = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, lt++) {
            const int buf = lt % nbuf, use = lt / nbuf;
            if (use >= 1) mbar_wait(acc_empty + buf, (use & 1) ^ 1);  // the epilogue drained this accumulator
            tc_fence_after();
            const uint32_t dacc = tmem + buf * 256;
            bool first = true;
            for (int cb = 0; cb < ncb; cb++) {
                for (int dyi = 0; dyi < 3; dyi++, ia++) {
                    const int sa = ia % NA;
                    mbar_wait(a_full + sa, (ia / NA) & 1);
                    for (int dxi = 0; dxi < 3; dxi++, ib++) {
                        const int sb = ib % NB;
                        mbar_wait(b_full + sb, (ib / NB) & 1);
                        tc_fence_after();
                        if (lane == 0) {
                            // tap (dy, dx): staging rows shifted by 1 + dx; the 4 MMAs of the K block walk planes 2kk, 2kk+1
                            const uint32_t a0 = abase + sa * A_SLOT + dxi * 16;
                            for (int j = 0; j < nsub; j++) {
#pragma unroll
                                for (int kk = 0; kk < 4; kk++) {
                                    const uint64_t ad = none_desc(a0 + 2 * kk * PLANE);
                                    const uint64_t bd = sw128_desc(bb + sb * L.bstage + j * bns * 128 + kk * 32);
                                    const uint32_t acc = (first && kk == 0) ? 0u : 1u;
                                    asm volatile(
                                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                                            dacc + j * bns),
                                        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                                }
                            }
                            mma_commit(b_empty + sb);
                            if (dxi == 2) mma_commit(a_empty + sa);
                            if (cb == ncb - 1 && dyi == 2 && dxi == 2) mma_commit(acc_full + buf);
                        }
                        first = false;
                        __syncwarp();
                    }
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue (warps 6-9)
        const int et = tid - EPI_WARP0 * 32, quarter = warp & 3, lr = quarter * 32 + lane;
        const EpiCtx e = make_epi(a, t);
        EpiTab tb;
        tb.bias = biastab;
        tb.b2 = biastab + bn;
        tb.mean = tb.rstd = tb.gamma = tb.beta = nullptr;
        int lt = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, lt++) {
            const int m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * bn;
            named_sync(1, 128);
            for (int c = et; c < bn; c += 128) {
                const bool ok = n0 + c < a.n;
                tb.bias[c] = ok && a.bias ? __ldg(a.bias + n0 + c) : 0.f;
                tb.b2[c] = ok && e.bias2 ? load_elem(e.bias2, a.bias2.dtype, n0 + c) : 0.f;
            }
            named_sync(1, 128);
            const int buf = lt % nbuf;
            mbar_wait(acc_full + buf, (lt / nbuf) & 1);
            tc_fence_after();
            const int r = m0 + lr;
            const int orow = r < a.m ? __ldg(a.d_rows + r) : -1;
            const uint32_t taddr = tmem + buf * 256 + ((uint32_t)(quarter * 32) << 16);
            for (int cb = 0; cb < bn; cb += 16) {
                uint32_t u[16];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
                      "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]),
                      "=r"(u[15])
                    : "r"(taddr + cb));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (orow < 0 || n0 + cb >= a.n) continue;
                float v[16];
#pragma unroll
                for (int j = 0; j < 16; j++) v[j] = __uint_as_float(u[j]);
                if (a.epi == FIS_EPI_STEP) row_epilogue<FIS_EPI_STEP>(a, e, tb, r, cb, n0, v);  // out conv
                else row_epilogue<FIS_EPI_NONE>(a, e, tb, r, cb, n0, v);
            }
            tc_fence_before();
            mbar_arrive(acc_empty + buf);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace halo
}  // namespace fis

// Halo-mode gathered conv on the persistent kernel: bf16 sources (16-byte rows), 64 | channels of
// every segment, bias (+ time bias) epilogue with a bf16 row-major output (the stacked step applies
// GroupNorm separately) or the out conv's latent step update, static TMA-addressable weights.
int fis_gemm_halo_ok(const fis_gemm_args* a) {
    static int off = getenv("FIS_HALO") && getenv("FIS_HALO")[0] == '0';
    if (off || !a->m_halo || a->a_mode != FIS_A_CONV3X3 || !a->rows || !a->d_rows || a->splits > 1) return 0;
    // epilogues: bias (+ time bias), or the out conv's latent step update (f32 latent rows)
    if ((a->epi != FIS_EPI_NONE && a->epi != FIS_EPI_STEP) || a->alpha != 1.0f || a->pre.ptr || a->pre2.ptr ||
        a->res.ptr || a->d_trans || a->n_split)
        return 0;
    if (a->epi == FIS_EPI_NONE && (a->d.dtype != FIS_BF16 || (a->d.ld % 8))) return 0;
    if (a->b.dtype != FIS_BF16 || a->b.step_stride || (a->b.ld % 8)) return 0;
    for (int i = 0; i < a->nsrc; i++) {
        const fis_src& s = a->src[i];
        if (s.c % 64 || s.fresh.dtype != FIS_BF16 || (s.fresh.ld % 8)) return 0;
        if (s.index && (s.cache.dtype != FIS_BF16 || (s.cache.ld % 8))) return 0;
    }
    return 1;
}

static int halo_bn(int n) {
    static int force = getenv("FIS_HALO_BN") ? atoi(getenv("FIS_HALO_BN")) : 0;
    if (force && n % force == 0) return force;
    for (int bn = 512; bn > 256; bn -= 32)
        if (n % bn == 0 && (bn / 2) % 16 == 0) return bn;
    for (int bn = 256; bn >= 64; bn -= 16)
        if (n % bn == 0) return bn;
    return n <= 256 ? (n + 15) & ~15 : 256;
}

int fis_gemm_halo_launch(const fis_gemm_args* a, cudaStream_t stream) {
    if (!fis_gemm_halo_ok(a)) return FIS_ERR_UNSUPPORTED;
    const int bn = halo_bn(a->n);
    const CUtensorMap* tm = fis_weight_map(a->b.ptr, a->n, a->k, a->b.ld, bn > 256 ? bn / 2 : bn);
    if (!tm) return FIS_ERR_UNSUPPORTED;
    const fis::halo::Layout L = fis::halo::layout(bn);
    static int configured = 0;
    if (configured < L.total) {
        if (cudaFuncSetAttribute(fis::halo::gemm_halo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - 1024) !=
            cudaSuccess)
            return FIS_ERR_UNSUPPORTED;
        configured = 227 * 1024 - 1024;
    }
    if (L.total > configured) return FIS_ERR_UNSUPPORTED;
    int sm = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, dev);
    const long long tiles = (long long)((a->m + 127) / 128) * ((a->n + bn - 1) / bn);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(tiles < sm ? tiles : sm));
    cfg.blockDim = dim3(fis::halo::THREADS);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = fis_pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fis::halo::gemm_halo_kernel, *a, *tm, bn) == cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
}
