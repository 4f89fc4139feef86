// Persistent 2-SM (CTA pair) tcgen05 GEMM for large M with TMA-staged A: dense 3x3 conv taps
// (4-D boxes, zero fill = padding) or contiguous rows.
//
//   D[r, n] = epi( sum_k A[r,k] * B[n,k] ),  bf16 operands, fp32 accumulation in TMEM.
//
// Why: the single-SM kernels (fis_gemm_big.cu) read BOTH operands from their own shared memory
// for every MMA and also receive every TMA byte there: at 128 x 256 x 16 per 128 cycles that is
// 12 KB of operand reads + 12 KB of TMA writes, ~190 B/cycle against a ~128 B/cycle port, which
// caps the dense convs of the stacked step at ~63% of the tensor peak. A CTA pair
// (tcgen05.mma.cta_group::2, M = 256) splits B between the two SMs: each SM stages its 128 A rows
// and HALF of the 256-wide B tile, the pair's tensor cores exchange the B halves, so per SM and
// MMA it is 8 KB of reads + 8 KB of writes.
//
// Roles (each CTA, 320 threads):
//   warp 4 (lane 0) : TMA producer: per K block its A rows {64 x 128} and its B half {64 x 128};
//                     completion is signalled on the LEADER's full barrier (.cta_group::2), the
//                     leader alone expects the pair's 64 KB.
//   warp 5          : TMEM (cta_group::2 allocation, 2 x 256 columns); in the leader (rank 0)
//                     lane 0 issues tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 16) and
//                     commits stage / accumulator barriers to BOTH CTAs (multicast).
//   warps 0-3, 6-9  : epilogue of this CTA's 128 rows: tcgen05.ld, fused row epilogue, stores;
//                     then one arrival on the leader's accumulator-empty barrier.
#include "fis_tc.cuh"
#include "fis_tma.cuh"
#include <cstdlib>

int fis_tma_a_encode(const fis_gemm_args* a, CUtensorMap* ta, CUtensorMap* ta2);
const CUtensorMap* fis_weight_map(const void* base, long long n, long long k, long long ld, int box);

namespace fis {
namespace pair {

using namespace fis::tc;

constexpr int THREADS = 320, TMA_WARP = 4, MMA_WARP = 5;
constexpr int BN = 256;                       // pair tile: 256 rows x 256 columns
constexpr int A_BYTES = BM * BK * 2;          // 16 KB: this CTA's 128 rows of the K block
constexpr int B_BYTES = (BN / 2) * BK * 2;    // 16 KB: this CTA's half of the B tile
constexpr int STAGE = A_BYTES + B_BYTES;
// OST (small K, plain row-major epilogue): 5 stages + two 16 KB output staging boxes for TMA stores
template <bool OST> struct Cfg {
    static constexpr int STAGES = OST ? 5 : 6;
};
constexpr int AM_ROWS = 1, AM_CONV = 2;
constexpr int STG_BYTES = 8 * 16 * 32 * 2;  // (reserved: the former per-warp V^T transpose tiles)
constexpr int TAIL = 15360;  // barriers (256) + epilogue tables (6 x BN floats) + reserved, 1 KB aligned
static_assert(256 + 6 * BN * 4 + STG_BYTES <= TAIL, "pair kernel tail");
template <bool OST> constexpr int smem_bytes() { return Cfg<OST>::STAGES * STAGE + TAIL + (OST ? 2 * 16384 : 0); }

FIS_DEV uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
FIS_DEV uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t d;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(addr), "r"(rank));
    return d;
}
FIS_DEV void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA loads of a CTA pair: data into this CTA's shared memory, completion on the barrier at the
// shared::cluster address bar (the leader's)
FIS_DEV void tma2d_pair(uint32_t dst, const void* tmap, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
FIS_DEV void tma4d_pair(uint32_t dst, const void* tmap, int c0, int c1, int c2, int c3, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4, %5}], [%6];" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}
// commit the leader's prior MMAs to the barrier at the same offset in both CTAs of the pair
FIS_DEV void commit_pair(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "h"((unsigned short)3)
                 : "memory");
}
FIS_DEV void tmem_ld16(uint32_t taddr, uint32_t* u) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
          "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <bool OST>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_pair_kernel(const fis_gemm_args a, const __grid_constant__ CUtensorMap tmap_b,
                     const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_a2,
                     const __grid_constant__ CUtensorMap tmap_d, int amode) {
    constexpr int STAGES = Cfg<OST>::STAGES;
    const int ls = ltr_begin(14);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = (uint64_t*)(smem + STAGES * STAGE);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;  // [2]
    uint64_t* acc_empty = acc_full + 2;   // [2]
    uint32_t* tmem_slot = (uint32_t*)(acc_empty + 2);
    float* tabs = (float*)(smem + STAGES * STAGE + 256);
    unsigned char* ostg = smem + STAGES * STAGE + TAIL;  // OST: two [128 x 64] bf16 SW128 boxes

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const int pair_id = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int tiles_n = (a.n + BN - 1) / BN, tiles_m = (a.m + 2 * BM - 1) / (2 * BM);
    const int ntiles = tiles_m * tiles_n;
    const int kblocks = (a.k + BK - 1) / BK;

    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(full + s, 1);   // used in the leader: its producer's expect_tx arrival
            mbar_init(empty + s, 1);  // the leader's MMA commit (multicast)
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(acc_full + b, 1);   // the leader's MMA commit (multicast)
            mbar_init(acc_empty + b, 2);  // leader: one arrival per CTA's drained epilogue
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == TMA_WARP && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_b) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_a) : "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // both CTAs' barriers initialised and TMEM allocated
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int t = cur_step(a.step);
    pdl_trigger();
    pdl_wait();
    ltr(ls, 2);

    if (warp == TMA_WARP) {
        // ------------------------------------------------------------ TMA producer (both CTAs)
        if (lane == 0) {
            const uint32_t sbase = smem_u32(smem);
            const int ow = a.out_w, ohw = a.out_h * a.out_w;
            const int cin0 = a.nsrc > 0 ? a.src[0].c : 0, cin = cin0 + (a.nsrc > 1 ? a.src[1].c : 0);
            int it = 0;
            for (int tile = pair_id; tile < ntiles; tile += npairs) {
                const int n0 = (tile % tiles_n) * BN;
                const int m0 = (tile / tiles_n) * 2 * BM + (int)rank * BM;  // this CTA's 128 rows
                const int img = amode == AM_CONV ? m0 / ohw : 0;
                const int y0 = amode == AM_CONV && ohw >= BM ? (m0 - img * ohw) / ow : 0;
                for (int kb = 0; kb < kblocks; kb++, it++) {
                    const int s = it % STAGES;
                    if (it >= STAGES) mbar_wait(empty + s, ((it / STAGES) & 1) ^ 1);
                    const uint32_t lbar = mapa(smem_u32(full + s), 0);
                    if (rank == 0)
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + s)),
                                     "r"((uint32_t)(2 * STAGE))
                                     : "memory");
                    const uint32_t sa = sbase + s * STAGE;
                    tma2d_pair(sa + A_BYTES, &tmap_b, kb * BK, n0 + (int)rank * (BN / 2), lbar);
                    if (amode == AM_ROWS) {
                        tma2d_pair(sa, &tmap_a, kb * BK, m0, lbar);
                    } else {
                        const int k0 = kb * BK, tap = k0 / cin;
                        int c = k0 - tap * cin;
                        const bool seg1 = c >= cin0;
                        c -= seg1 ? cin0 : 0;
                        tma4d_pair(sa, seg1 ? &tmap_a2 : &tmap_a, c, tap % 3 - 1, y0 + tap / 3 - 1, img, lbar);
                    }
                }
            }
        }
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------------------ MMA issuer (leader only)
        if (rank == 0) {
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                   ((uint32_t)((2 * BM) >> 4) << 24);
            const uint32_t sbase = smem_u32(smem);
            int it = 0, lt = 0;
            for (int tile = pair_id; tile < ntiles; tile += npairs, lt++) {
                const int buf = lt & 1, use = lt >> 1;
                if (use >= 1) mbar_wait(acc_empty + buf, (use & 1) ^ 1);  // both CTAs drained this buffer
                tc_fence_after();
                const uint32_t dt = tmem + buf * BN;
                for (int kb = 0; kb < kblocks; kb++, it++) {
                    const int s = it % STAGES;
                    mbar_wait(full + s, (it / STAGES) & 1);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t sa = sbase + s * STAGE, sb = sa + A_BYTES;
#pragma unroll
                        for (int kk = 0; kk < BK / 16; kk++) {
                            const uint64_t ad = sw128_desc(sa + kk * 32), bd = sw128_desc(sb + kk * 32);
                            const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
                            asm volatile(
                                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
                                "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                        }
                        commit_pair(empty + s);
                        if (kb == kblocks - 1) commit_pair(acc_full + buf);
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue (warps 0-3, 6-9)
        const int grp = warp < TMA_WARP ? 1 : 0;
        const int et = grp ? tid + 128 : tid - 6 * 32;  // 0..255
        const int quarter = warp & 3;
        const int lr = quarter * 32 + lane;
        const EpiCtx e = make_epi(a, t);
        const bool fast = a.epi == FIS_EPI_NONE && a.alpha == 1.0f && !e.pre && !e.pre2 && !e.bias2 && !e.lat &&
                          !a.d_rows && !a.d_trans && a.d.dtype == FIS_BF16 && (a.d.ld % 8) == 0 &&
                          (((uintptr_t)e.d) & 15) == 0 && (!e.res || (a.res.ld % 8) == 0);
        // fused QKV: the V^T part (n >= n_split) goes transposed to d2 through a per-warp staging tile
        const bool tfast = fast && !e.res && a.n_split > 0 && a.d2_trans && a.d2.dtype == FIS_BF16 &&
                           (a.d2.ld % 8) == 0 && (((uintptr_t)e.d2) & 15) == 0;
        const int nrow_end = a.n_split > 0 ? a.n_split : a.n;  // row-major columns
        const bool ost = OST && fast && (a.n_split % 64) == 0;
        int nbox = 0;
        EpiTab tb;
        tb.mean = tabs;
        tb.rstd = tb.mean + BN;
        tb.bias = tb.rstd + BN;
        tb.b2 = tb.bias + BN;
        tb.gamma = tb.b2 + BN;
        tb.beta = tb.gamma + BN;
        const uint32_t leader_empty0 = mapa(smem_u32(acc_empty), 0);
        int lt = 0;
        for (int tile = pair_id; tile < ntiles; tile += npairs, lt++) {
            const int n0 = (tile % tiles_n) * BN;
            const int m0 = (tile / tiles_n) * 2 * BM + (int)rank * BM;
            asm volatile("bar.sync 1, 256;" ::: "memory");  // previous tile's table reads done
            for (int c = et; c < BN; c += 256) {
                const int n = n0 + c;
                const bool ok = n < a.n;
                tb.bias[c] = ok && a.bias ? __ldg(a.bias + n) : 0.f;
                tb.b2[c] = ok && e.bias2 ? load_elem(e.bias2, a.bias2.dtype, n) : 0.f;
                tb.gamma[c] = 0.f;
                tb.beta[c] = 0.f;
                if (a.epi == FIS_EPI_GN_SILU && ok) {
                    const int g = n / e.cpg;
                    const float rstd = (float)(1.0 / sqrt((double)e.var[g] + (double)a.eps));
                    const float scale = rstd * __ldg(a.gamma + n);
                    tb.mean[c] = scale;
                    tb.rstd[c] = fmaf(-e.mean[g], scale, __ldg(a.beta + n));
                } else {
                    tb.mean[c] = 0.f;
                    tb.rstd[c] = 0.f;
                }
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
            const int buf = lt & 1;
            mbar_wait(acc_full + buf, (lt >> 1) & 1);
            tc_fence_after();
            const uint32_t taddr = tmem + buf * BN + ((uint32_t)(quarter * 32) << 16);
            const int r = m0 + lr;
            for (int bx = 0; bx < BN / 64; bx++) {
            // OST: a 64-column box of plain row-major outputs goes through a SW128 staging box and
            // one TMA store instead of 32-byte row stores per thread
            const bool sbox = ost && n0 + bx * 64 + 64 <= nrow_end;
            unsigned char* sb = ostg + (nbox & 1) * 16384;
            if (sbox) {
                if (et == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // box nbox - 2 read
                asm volatile("bar.sync 1, 256;" ::: "memory");
            }
            for (int h = 0; h < 2; h++) {  // the two warp groups take alternate 16-column chunks
                const int cb = bx * 64 + 16 * grp + 32 * h;
                uint32_t u[16];
                tmem_ld16(taddr + cb, u);
                const int n = n0 + cb;
                if (sbox) {
                    float v[16];
#pragma unroll
                    for (int j = 0; j < 16; j++) v[j] = __fadd_rn(__uint_as_float(u[j]), tb.bias[cb + j]);
                    if (e.res && r < a.m) {
                        float q[16];
                        load_row16(e.res, a.res.dtype, (long long)r * a.res.ld + n, 16, q);
#pragma unroll
                        for (int j = 0; j < 16; j++) v[j] = __fadd_rn(v[j], q[j]);
                    }
                    uint4 o[2];
                    __nv_bfloat162* hh = (__nv_bfloat162*)o;
#pragma unroll
                    for (int j = 0; j < 8; j++) hh[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
                    const int un = (cb & 63) >> 3;
                    *(uint4*)(sb + sw128_off(lr, un)) = o[0];
                    *(uint4*)(sb + sw128_off(lr, un + 1)) = o[1];
                    continue;
                }
                if (tfast && n >= a.n_split && n + 16 <= a.n) {  // warp-uniform: V^T chunk
                    // V^T[dn + j][r]: for each j the warp's 32 rows are 64 contiguous bytes -- direct
                    // 2-byte stores, coalesced per j (the shared-memory transpose round trip it replaces
                    // was the epilogue's top stall: R = 64 L0 / L1 / L2 QKV 36 / 25 / 77 -> 28.5 / 22 / 72.5 us)
                    if (r < a.m) {
                        __nv_bfloat16* dst = (__nv_bfloat16*)e.d2 + (long long)(n - a.n_split) * a.d2.ld + r;
#pragma unroll
                        for (int j = 0; j < 16; j++)
                            dst[(long long)j * a.d2.ld] = __float2bfloat16_rn(__fadd_rn(__uint_as_float(u[j]), tb.bias[cb + j]));
                    }
                    continue;
                }
                if (r >= a.m || n >= a.n) continue;
                float v[16];
#pragma unroll
                for (int j = 0; j < 16; j++) v[j] = __uint_as_float(u[j]);
                if (fast && n + 16 <= nrow_end) {
#pragma unroll
                    for (int j = 0; j < 16; j++) v[j] = __fadd_rn(v[j], tb.bias[cb + j]);
                    if (e.res) {
                        float q[16];
                        load_row16(e.res, a.res.dtype, (long long)r * a.res.ld + n, 16, q);
#pragma unroll
                        for (int j = 0; j < 16; j++) v[j] = __fadd_rn(v[j], q[j]);
                    }
                    uint4 o[2];
                    __nv_bfloat162* h = (__nv_bfloat162*)o;
#pragma unroll
                    for (int j = 0; j < 8; j++) h[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
                    uint4* dp = (uint4*)((__nv_bfloat16*)e.d + (long long)r * a.d.ld + n);
                    dp[0] = o[0];
                    dp[1] = o[1];
                } else {
                    row_epilogue_any(a, e, tb, r, cb, n0, v);
                }
            }
            if (sbox) {
                fence_async_smem();  // generic-proxy box writes -> the TMA store
                asm volatile("bar.sync 1, 256;" ::: "memory");
                if (et == 0) {
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tmap_d),
                                 "r"(n0 + bx * 64), "r"(m0), "r"(smem_u32(sb))
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                nbox++;
            }
            }
            tc_fence_before();
            asm volatile("bar.sync 1, 256;" ::: "memory");  // every epilogue thread of this CTA read the buffer
            if (et == 0)
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                 leader_empty0 + (uint32_t)(buf * 8))
                             : "memory");
        }
        if (OST && et == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging read before exit
    }
    ltr(ls, 7);
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // the peer's MMAs / remote arrivals are done before TMEM and shared memory go away
    if (warp == MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace pair
}  // namespace fis

static long long g_pair_launched = 0;
extern "C" long long fis_gemm_pair_launch_count(void) { return g_pair_launched; }

static int pair_sms() {
    static int n = 0;
    if (n <= 0) n = fis_device_sm_count();
    return n > 0 ? n : 148;
}

// The pair kernel takes large-M GEMMs whose A the TMA can stage (dense conv taps / contiguous rows),
// static bf16 weights, no split-K / transposed outputs (a fused QKV's V^T half is fine), when its
// 256 x 256 tiles need no more time than the single-SM kernel's tiles (rounds of tiles x width at the
// measured ~0.92 vs ~0.55 of the tensor peak: ncu tensor-pipe utilisation of the 64-request step,
// profiles/r02/ncu_gemms_R64_*.csv).
int fis_gemm_pair_ok(const fis_gemm_args* a, int single_bn) {
    // FIS_PAIR=0 disables, =2 forces (read per call: tests switch it; fis_gemm runs at capture time)
    const char* env = getenv("FIS_PAIR");
    const int off = env && env[0] == '0', force = env && env[0] == '2';
    if (off || a->splits > 1 || a->b.step_stride || a->b.dtype != FIS_BF16 || (a->b.ld % 8) || a->d_trans || a->rows ||
        a->n < 256)
        return 0;
    // fused QKV (V^T to d2): 16-column chunks never straddle the split
    if (a->n_split > 0 && (a->n_split % 16 || !a->d2_trans)) return 0;
    CUtensorMap ta, ta2;
    if (!fis_tma_a_encode(a, &ta, &ta2)) return 0;
    const long long sms = pair_sms();
    const long long t2 = (long long)((a->m + 255) / 256) * ((a->n + 255) / 256);
    const double c2 = (double)((t2 + sms / 2 - 1) / (sms / 2)) * 256 / 0.92;
    double c1 = 0;
    for (int bn : {single_bn, 320}) {  // the single-SM kernel's 256-wide tiles or 320-wide (two MMAs)
        if (bn == 320 && a->n % 320) continue;
        const long long t1 = (long long)((a->m + 127) / 128) * ((a->n + bn - 1) / bn);
        const double c = (double)((t1 + sms - 1) / sms) * bn / 0.55;
        if (c1 == 0 || c < c1) c1 = c;
    }
    return force || c2 < c1;
}

// OST variant for small-K GEMMs with a plain bf16 row-major epilogue (FIS_PAIR_OST: 0 off, 2 any K)
static bool pair_ost(const fis_gemm_args* a, CUtensorMap* td) {
    static int mode = getenv("FIS_PAIR_OST") ? atoi(getenv("FIS_PAIR_OST")) : 1;
    if (mode == 0 || (mode == 1 && a->k > 640)) return false;
    if (a->epi != FIS_EPI_NONE || a->alpha != 1.0f || a->pre.ptr || a->pre2.ptr || a->bias2.ptr || a->lat.ptr ||
        a->d_rows || a->d_trans || a->d.dtype != FIS_BF16 || a->d.step_stride || (a->d.ld % 8) ||
        (a->res.ptr && ((a->res.ld % 8) || a->res.step_stride)) || (a->n_split % 64))
        return false;
    const int ncols = a->n_split > 0 ? a->n_split : a->n;
    return encode_2d(td, a->d.ptr, a->m, ncols, a->d.ld, 128);
}

int fis_gemm_pair_launch(const fis_gemm_args* a, cudaStream_t stream) {
    CUtensorMap ta, ta2, td;
    std::memset(&ta, 0, sizeof(ta));
    std::memset(&ta2, 0, sizeof(ta2));
    std::memset(&td, 0, sizeof(td));
    const int amode = fis_tma_a_encode(a, &ta, &ta2);
    if (!amode) return FIS_ERR_UNSUPPORTED;
    const CUtensorMap* tm = fis_weight_map(a->b.ptr, a->n, a->k, a->b.ld, fis::pair::BN / 2);
    if (!tm) return FIS_ERR_UNSUPPORTED;
    const bool ost = pair_ost(a, &td);
    static bool configured = false;
    if (!configured) {
        if (cudaFuncSetAttribute(fis::pair::gemm_pair_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 fis::pair::smem_bytes<false>() + 1024) != cudaSuccess ||
            cudaFuncSetAttribute(fis::pair::gemm_pair_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 fis::pair::smem_bytes<true>() + 1024) != cudaSuccess)
            return FIS_ERR_UNSUPPORTED;
        configured = true;
    }
    const long long tiles = (long long)((a->m + 255) / 256) * ((a->n + 255) / 256);
    const int npairs = (int)(tiles < pair_sms() / 2 ? tiles : pair_sms() / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * npairs);
    cfg.blockDim = dim3(fis::pair::THREADS);
    cfg.dynamicSmemBytes = (ost ? fis::pair::smem_bytes<true>() : fis::pair::smem_bytes<false>()) + 1024;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = fis_pdl_enabled() ? 2 : 1;
    const cudaError_t e = ost ? cudaLaunchKernelEx(&cfg, fis::pair::gemm_pair_kernel<true>, *a, *tm, ta, ta2, td, amode)
                              : cudaLaunchKernelEx(&cfg, fis::pair::gemm_pair_kernel<false>, *a, *tm, ta, ta2, td, amode);
    if (e != cudaSuccess) return FIS_ERR_LAUNCH;
    g_pair_launched++;
    return FIS_OK;
}

FIS_LTR_SETTER(fis_ltr_set_pair)
