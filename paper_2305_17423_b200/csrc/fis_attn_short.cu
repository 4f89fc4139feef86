// Short-run attention on tcgen05 (sm_100a): every key run <= 256 keys -- the stacked step's cross
// attention (77-token prompts, sparse.py:303-338/352-361) and short self-attention runs (the
// 8x8 and 16x16 levels, sparse.py:265-300) -- as ONE persistent kernel per call:
//
//   out[r, :] = res[r, :] + softmax(Q K^T * scale)[r, :] V        (unet.py:279-293, 555-566)
//
// fis_attn's general kernel gives every (query tile, 256-column value slice) its own CTA: for one
// key block that is a latency chain per CTA (load Q, S, softmax, P.V, then a residual + store
// epilogue on LDGs) with one CTA per SM, so the stacked cross attention ran at 15-20% of the HBM
// roofline it is bound by (q + res + out bytes). Here a CTA loops over work units (segment, 128-
// query tile, group of 128-column value slices) and overlaps the stages of consecutive units:
//
//   TMA producer    : per unit the d/64 chunks Q {128 x 64} + K {KP x 64} (KP = run
//                     length rounded to 16), then per value slice the V^T chunks {128 x 64 keys}
//   MMA issuer      : S = Q K^T (M = 128, N = KP) into TMEM columns 0..KP, then per
//                     slice O_s = P V_s (K = KP) into one of three 128-column TMEM buffers
//   warps 0-3       : softmax, thread = query row: statistics + normalised bf16 P into a SW128
//                     shared tile (the S buffer is released as soon as P is written, so S of the
//                     next unit overlaps this unit's P.V and epilogue)
//   warps 4-11      : epilogue, thread = (row, 64-column half): O (tcgen05.ld) + the staged
//                     residual tile -> bf16, written back into the tile in place
//   warp 14         : residual loads + output stores over a ring of NEB staging tiles: TMA loads
//                     of the residual tiles NEB - 1 jobs ahead, TMA stores of each finished tile in
//                     whole 8-row groups (1 KB swizzle atoms -- rows of a neighbouring run are never
//                     written), 16-byte row stores for a run's < 8 trailing rows
//   warp 12 (lane 0): TMA producer, warp 13: MMA issuer (above)
//
// Numerics follow fis_attn's one-block path exactly (same log2-domain statistics over 32-column
// chunks, P = 2^(s*scale*log2e - m - log2 l) rounded to bf16, fp32 accumulation, out = bf16(O + res)).
#include "fis_attn.cuh"
#include "fis_tma.cuh"
#include <cstdlib>
#include <cstring>

namespace fis {
namespace attn_short {

using namespace fis::attn;

constexpr int THREADS = 480, EPI_WARP0 = 4, TMA_WARP = 12, MMA_WARP = 13, STORE_WARP = 14;
constexpr int CH = 16384;       // one SW128 chunk: 128 rows x 128 B
constexpr int MAX_RUNS = 127;   // runs per call (tile-count prefix in shared memory)
// Per key-run bound KMAX:
//   128: value slices of SW = 128 columns; stages of 32 KB (Q chunk 16 KB + K chunk <= 16 KB, or two
//        V^T chunks {64 keys x 128}); P tile 32 KB; S in TMEM columns 0-127, three 128-column O buffers
//   256: (129-256-key runs: the stacked step's 16x16-level self attention) SW = 64; two 48 KB
//        stages (Q 16 KB + K <= 32 KB, or four V^T chunks {64 keys x 64}); P tile 64 KB; S in
//        columns 0-255, four 64-column O buffers
// Residual / output staging: three tiles of 128 rows x SW columns.
template <int KMAX> struct KC;
template <> struct KC<128> {
    static constexpr int SW = 128, STAGES = 3, STAGE = 32768, PT = 32768, NOB = 3, NEB = 3;
};
template <> struct KC<256> {
    static constexpr int SW = 64, STAGES = 2, STAGE = 49152, PT = 65536, NOB = 4, NEB = 3;
};
template <int KMAX> constexpr int smem_bytes() {
    return KC<KMAX>::STAGES * KC<KMAX>::STAGE + KC<KMAX>::PT + KC<KMAX>::NEB * KC<KMAX>::SW * 256 + 1024 + 256 +
           4 * (MAX_RUNS + 1);
}

struct Unit {
    int m0, rows, k0, nk, s0, s1;
};

// Work schedule: the real query tiles of all runs, numbered run by run (cum[s] = tiles of runs
// before s, in shared memory), times G slice groups; unit u = tile (u / G), slice group (u % G).
// Numbering only real tiles keeps the round-robin over the persistent CTAs balanced whatever the
// run lengths (a padded [run][max tiles] grid left most CTAs of ragged calls one unit and a few two).
struct Sched {
    const int* cum;
    int nseg, G, ns, nunits;
};

FIS_DEV void run_bounds(const fis_attn_args& a, int sg, int& qb, int& qe, int& kb, int& ke) {
    qb = 0, qe = a.m, kb = 0, ke = a.n_keys;
    if (a.nseg > 0) {
        qb = __ldg(a.q_seg + 2 * sg);
        qe = __ldg(a.q_seg + 2 * sg + 1);
        kb = __ldg(a.k_seg + 2 * sg);
        ke = __ldg(a.k_seg + 2 * sg + 1);
    }
}

FIS_DEV bool unit_of(const fis_attn_args& a, const Sched& sc, int u, Unit& x) {
    const int g = u % sc.G, r = u / sc.G;
    int lo = 0, hi = sc.nseg;  // the run holding tile r: last s with cum[s] <= r
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (sc.cum[mid] <= r) lo = mid;
        else hi = mid;
    }
    int qb, qe, kb, ke;
    run_bounds(a, lo, qb, qe, kb, ke);
    x.m0 = qb + (r - sc.cum[lo]) * 128;
    x.rows = min(128, qe - x.m0);
    x.k0 = kb;
    x.nk = ke - kb;  // <= KP (the host sizes KP from the longest run)
    x.s0 = g * sc.ns / sc.G;
    x.s1 = (g + 1) * sc.ns / sc.G;
    return x.rows > 0 && x.nk > 0 && x.s1 > x.s0;
}

// advance u (stepping by the grid) to the next non-empty unit; false when the CTA has none left
FIS_DEV bool seek_unit(const fis_attn_args& a, const Sched& sc, int& u, Unit& x) {
    for (; u < sc.nunits; u += gridDim.x)
        if (unit_of(a, sc, u, x)) return true;
    return false;
}

template <int KMAX>
__global__ void __launch_bounds__(THREADS, 1)
    attn_short_kernel(const fis_attn_args a, const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tq16,
                      const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                      const __grid_constant__ CUtensorMap tr, const __grid_constant__ CUtensorMap to,
                      const __grid_constant__ CUtensorMap to8, int KP, int G_req) {
    constexpr int SW = KC<KMAX>::SW, STAGES = KC<KMAX>::STAGES, STAGE = KC<KMAX>::STAGE, PT = KC<KMAX>::PT;
    constexpr int NOB = KC<KMAX>::NOB, NEB = KC<KMAX>::NEB, EBUF = SW * 256;
    constexpr uint32_t OCOL = KMAX;  // TMEM: S in columns [0, KMAX), O buffer b at OCOL + b * SW
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* ptile = smem + STAGES * STAGE;
    unsigned char* ebuf = ptile + PT;
    uint64_t* full = (uint64_t*)(ebuf + NEB * EBUF);
    uint64_t* empty = full + STAGES;
    uint64_t* s_full = empty + STAGES;
    uint64_t* s_free = s_full + 1;
    uint64_t* p_full = s_free + 1;
    uint64_t* p_free = p_full + 1;
    uint64_t* o_full = p_free + 1;     // [NOB]
    uint64_t* o_free = o_full + NOB;   // [NOB]
    uint64_t* r_full = o_free + NOB;   // [NEB] residual tile landed
    uint64_t* staged = r_full + NEB;   // [NEB] bf16(O + residual) written back (epilogue threads)
    uint32_t* tmem_slot = (uint32_t*)(staged + NEB);
    int* cum = (int*)(ebuf + NEB * EBUF + 256);  // [MAX_RUNS + 1]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int dch = a.d / 64, ns = (a.dv + SW - 1) / SW;
    __shared__ int ls_sh;  // launch-trace slot (profiling builds; -1 otherwise)
    if (tid == 0) {
        ls_sh = ltr_begin(13);
        for (int i = 0; i < STAGES; i++) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
        }
        mbar_init(s_full, 1);
        mbar_init(s_free, 128);
        mbar_init(p_full, 128);
        mbar_init(p_free, 1);
        for (int b = 0; b < NOB; b++) {
            mbar_init(o_full + b, 1);
            mbar_init(o_free + b, 256);
        }
        for (int b = 0; b < NEB; b++) {
            mbar_init(r_full + b, 1);
            mbar_init(staged + b, 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == TMA_WARP && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tq) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tq16) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tk) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tv) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tr) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&to) : "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    const int nseg = a.nseg > 0 ? a.nseg : 1;
    if (warp == 0) {  // tile-count prefix over the runs (plan data: safe before the dependency wait)
        const int per = (nseg + 31) >> 5;  // <= 4
        int loc[4], sum = 0;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int sg = lane * per + i;
            loc[i] = 0;
            if (i < per && sg < nseg) {
                int qb, qe, kb, ke;
                run_bounds(a, sg, qb, qe, kb, ke);
                loc[i] = (qe > qb && ke > kb) ? (qe - qb + 127) >> 7 : 0;
            }
            sum += loc[i];
        }
        int incl = sum;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        int ex = incl - sum;
        for (int i = 0; i < per; i++) {
            const int sg = lane * per + i;
            if (sg < nseg) cum[sg] = ex;
            ex += loc[i];
        }
        if (lane == 31) cum[nseg] = incl;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    Sched sc;
    sc.cum = cum;
    sc.nseg = nseg;
    sc.ns = ns;
    {
        const int total = cum[nseg];
        int G = G_req > 0 ? G_req : (total > 0 ? (int)gridDim.x / total : 1);
        sc.G = max(1, min(G, ns));
        sc.nunits = total * sc.G;
    }
    const int t = cur_step(a.step);  // host-written before the step
    // this CTA's first unit: the segment tables are plan data (no kernel of the step writes them),
    // so they are decoded while the previous kernel drains
    int u0 = blockIdx.x;
    Unit x0;
    const bool have0 = seek_unit(a, sc, u0, x0);
    if (warp == TMA_WARP && lane == 0 && have0)  // the first unit's key rows into L2 (harmless if a
        for (int kc = 0; kc < dch; kc++)          // predecessor still writes them: L2 is coherent)
            tma_prefetch2d(&tk, kc * 64, x0.k0);
    pdl_trigger();
    pdl_wait();
    if (tid == 0) ltr(ls_sh, 1);

    if (warp == TMA_WARP) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            const uint32_t sbase = smem_u32(smem);
            const int nvc = (KP + 63) / 64;
            int it = 0, u = u0;
            Unit x = x0;
            for (bool have = have0; have; u += gridDim.x, have = seek_unit(a, sc, u, x)) {
                // a partial tile loads only its valid rows (16-row boxes): the MMA's other rows are
                // don't-care (rows are independent through S, P and O, and never stored)
                const int q16 = x.rows > 112 ? 8 : (x.rows + 15) >> 4;
                for (int kc = 0; kc < dch; kc++) {
                    const int st = it % STAGES;
                    if (it >= STAGES) mbar_wait(empty + st, ((it / STAGES) & 1) ^ 1);
                    arrive_expect_tx(full + st, (uint32_t)(q16 * 2048 + KP * 128));
                    if (q16 == 8) {
                        tma2d(sbase + st * STAGE, &tq, kc * 64, x.m0, full + st);
                    } else {
                        for (int g = 0; g < q16; g++) tma2d(sbase + st * STAGE + g * 2048, &tq16, kc * 64, x.m0 + g * 16, full + st);
                    }
                    tma2d(sbase + st * STAGE + CH, &tk, kc * 64, x.k0, full + st);
                    it++;
                }
                for (int s = x.s0; s < x.s1; s++) {
                    const int st = it % STAGES;
                    if (it >= STAGES) mbar_wait(empty + st, ((it / STAGES) & 1) ^ 1);
                    arrive_expect_tx(full + st, (uint32_t)(nvc * SW * 128));
                    for (int h = 0; h < nvc; h++) tma2d(sbase + st * STAGE + h * (SW * 128), &tv, x.k0 + h * 64, s * SW, full + st);
                    it++;
                }
            }
        }
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t sbase = smem_u32(smem), pbase = smem_u32(ptile);
        const uint32_t id_s = idesc_bf16(128, KP);
        const int ksteps = KP / 16;
        int it = 0, nu = 0, job = 0, u = u0;
        Unit x = x0;
        for (bool have = have0; have; u += gridDim.x, have = seek_unit(a, sc, u, x)) {
            if (nu >= 1) mbar_wait(s_free, (nu - 1) & 1);  // the softmax has read the previous S
            tc_fence_after();
            for (int kc = 0; kc < dch; kc++) {
                const int st = it % STAGES;
                mbar_wait(full + st, (it / STAGES) & 1);
                tc_fence_after();
                if (it == 0 && lane == 0) ltr(ls_sh, 9);
                if (lane == 0) {
                    const uint32_t sa = sbase + st * STAGE, sk = sa + CH;
#pragma unroll
                    for (int kk = 0; kk < 4; kk++)
                        mma_bf16(tmem, sw128_desc(sa + kk * 32), sw128_desc(sk + kk * 32), id_s, (kc | kk) ? 1u : 0u);
                    mma_commit(empty + st);
                    if (kc == dch - 1) mma_commit(s_full);
                }
                __syncwarp();
                it++;
            }
            mbar_wait(p_full, nu & 1);  // P of this unit in the shared tile
            tc_fence_after();
            for (int s = x.s0; s < x.s1; s++) {
                const int b = job % NOB;
                if (job >= NOB) mbar_wait(o_free + b, ((job / NOB) & 1) ^ 1);  // epilogue drained buffer b
                const int st = it % STAGES;
                mbar_wait(full + st, (it / STAGES) & 1);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t sv = sbase + st * STAGE;
                    const uint32_t id_o = idesc_bf16(128, min(SW, a.dv - s * SW));
                    for (int kk = 0; kk < ksteps; kk++) {
                        const uint32_t offp = (uint32_t)((kk >> 2) * CH + (kk & 3) * 32);
                        const uint32_t offv = (uint32_t)((kk >> 2) * (SW * 128) + (kk & 3) * 32);
                        mma_bf16(tmem + OCOL + b * SW, sw128_desc(pbase + offp), sw128_desc(sv + offv), id_o,
                                 kk ? 1u : 0u);
                    }
                    mma_commit(empty + st);
                    mma_commit(o_full + b);
                    if (s == x.s1 - 1) mma_commit(p_free);  // every P.V of this unit has read P
                }
                __syncwarp();
                it++;
                job++;
            }
            nu++;
        }
    } else if (warp < EPI_WARP0) {
        // ------------------------------------------------------------ softmax (warps 0-3)
        const int lr = tid;
        const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
        const float sl = a.scale * 1.4426950408889634f;
        float v[32];
        int nu = 0, u = u0;
        Unit x = x0;
        for (bool have = have0; have; u += gridDim.x, have = seek_unit(a, sc, u, x)) {
            mbar_wait(s_full, nu & 1);
            tc_fence_after();
            if (nu == 0 && tid == 0) ltr(ls_sh, 2);
            float mrow = -INFINITY, lrow = 0.f;
#pragma unroll 1
            for (int cb = 0; cb < KP; cb += 32) {
                tmem_ld32(trow + cb, v);
                const int lim = x.nk - cb;
                float cm = -INFINITY;
                if (lim >= 32) {
#pragma unroll
                    for (int q = 0; q < 32; q++) cm = fmaxf(cm, v[q]);
                } else {
#pragma unroll
                    for (int q = 0; q < 32; q++)
                        if (q < lim) cm = fmaxf(cm, v[q]);
                }
                const float mn = fmaxf(mrow, cm * sl);
                float add = 0.f;
                if (lim >= 32) {
#pragma unroll
                    for (int q = 0; q < 32; q++) add += ex2(fmaf(v[q], sl, -mn));
                } else {
#pragma unroll
                    for (int q = 0; q < 32; q++)
                        if (q < lim) add += ex2(fmaf(v[q], sl, -mn));
                }
                lrow = (mrow == -INFINITY ? 0.f : lrow * ex2(mrow - mn)) + add;
                mrow = mn;
            }
            const float off = mrow + __log2f(lrow);
            if (nu >= 1) mbar_wait(p_free, (nu - 1) & 1);  // the previous unit's P.V MMAs are done with P
#pragma unroll 1
            for (int cb = 0; cb < KP; cb += 32) {
                tmem_ld32(trow + cb, v);
                const int lim = x.nk - cb;
                unsigned char* pt = ptile + (cb >> 6) * CH;
#pragma unroll
                for (int u4 = 0; u4 < 4; u4++) {
                    uint4 pk;
                    __nv_bfloat162* h = (__nv_bfloat162*)&pk;
#pragma unroll
                    for (int e2 = 0; e2 < 4; e2++) {
                        const int q0 = 8 * u4 + 2 * e2;
                        const float p0 = q0 < lim ? ex2(fmaf(v[q0], sl, -off)) : 0.f;
                        const float p1 = q0 + 1 < lim ? ex2(fmaf(v[q0 + 1], sl, -off)) : 0.f;
                        h[e2] = __floats2bfloat162_rn(p0, p1);
                    }
                    *(uint4*)(pt + sw128_off(lr, ((cb & 63) >> 3) + u4)) = pk;
                }
            }
            tc_fence_before();
            mbar_arrive(s_free);  // S fully read
            fence_async_smem();   // generic-proxy P writes -> tensor-core reads
            mbar_arrive(p_full);
            if (nu == 0 && tid == 0) ltr(ls_sh, 3);
            nu++;
        }
    } else if (warp == STORE_WARP) {
        // ------------------------------------------------------------ residual loads + output stores
        // Job = (unit, slice). The NEB staging tiles form a ring: job j's residual tile is TMA-loaded
        // into tile j % NEB; the epilogue warps overwrite it in place with bf16(O + residual) and
        // arrive on staged[j % NEB]; this warp then TMA-stores the tile's whole 8-row groups (1 KB
        // swizzle atoms: rows of a neighbouring run are never written), writes the < 8 trailing rows
        // with 16-byte stores, and recycles the tile of job j - 1 (its stores have read it by now)
        // for the residual of job j - 1 + NEB. The store / recycle latency is off the epilogue's path.
        const bool tma_out = a.out.step_stride == 0;  // else the output moves with the step: row stores
        char* ob = ref_base(a.out, t);
        const uint32_t ebase = smem_u32(ebuf);
        auto advance = [&](int& uu, int& ss, Unit& xx) {  // next job after (uu, ss); false at the end
            if (++ss < xx.s1) return true;
            uu += gridDim.x;
            if (!seek_unit(a, sc, uu, xx)) return false;
            ss = xx.s0;
            return true;
        };
        auto load_res = [&](const Unit& xx, int ss, int b) {
            const int nbox = min(SW, a.dv - ss * SW) / 64;
            arrive_expect_tx(r_full + b, (uint32_t)(nbox * CH));
            for (int bx = 0; bx < nbox; bx++)
                tma2d(ebase + b * EBUF + bx * CH, &tr, ss * SW + bx * 64, xx.m0, r_full + b);
        };
        int u = u0, s = have0 ? x0.s0 : 0;
        Unit x = x0;
        bool have = have0;
        int lu = u, lsl = s;  // residual-load cursor
        Unit lx = x;
        bool lhave = have;
        if (lane == 0)
            for (int i = 0; lhave && i < NEB; i++) {
                load_res(lx, lsl, i);
                lhave = advance(lu, lsl, lx);
            }
        __syncwarp();
        int job = 0;
        while (have) {
            const int eb_i = job % NEB;
            const unsigned char* eb = ebuf + eb_i * EBUF;
            const uint32_t ebs = ebase + eb_i * EBUF;
            const int w = min(SW, a.dv - s * SW), nbox = w / 64;
            mbar_wait(staged + eb_i, (job / NEB) & 1);
            const int g8 = tma_out ? (x.rows >> 3) : 0;
            if (lane == 0) {
                for (int bx = 0; bx < nbox; bx++) {
                    if (g8 == 16) {
                        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&to),
                                     "r"(s * SW + bx * 64), "r"(x.m0), "r"(ebs + bx * CH)
                                     : "memory");
                    } else {
                        for (int g = 0; g < g8; g++)
                            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&to8),
                                         "r"(s * SW + bx * 64), "r"(x.m0 + g * 8), "r"(ebs + bx * CH + g * 1024)
                                         : "memory");
                    }
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");  // (possibly empty)
            }
            const int r0 = g8 * 8, upr = w >> 3, total = (x.rows - r0) * upr;
            if (total > 0) {
                const int sh = w == 128 ? 4 : 3;
                __nv_bfloat16* orow = (__nv_bfloat16*)ob + (long long)(x.m0 + r0) * a.out.ld + s * SW;
                for (int i = lane; i < total; i += 32) {
                    const int r = i >> sh, un = i & (upr - 1);
                    const uint4 val = *(const uint4*)(eb + (un >> 3) * CH + sw128_off(r0 + r, un & 7));
                    *(uint4*)(orow + (long long)r * a.out.ld + un * 8) = val;
                }
                fence_async_smem();  // generic reads of this tile before a later TMA write into it
            }
            __syncwarp();
            if (lane == 0 && job >= 1 && lhave) {  // recycle job - 1's tile
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                load_res(lx, lsl, (job - 1) % NEB);
                lhave = advance(lu, lsl, lx);
            }
            __syncwarp();
            have = advance(u, s, x);
            job++;
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // tiles read before exit
        if (lane == 0) ltr(ls_sh, 8);
    } else {
        // ------------------------------------------------------------ epilogue (warps 4-11)
        // warps 4-7 take the slice's columns 0-63, warps 8-11 columns 64-127 (one SW128 box each);
        // thread = row (warp % 4 selects the TMEM lane quarter): O (tcgen05.ld) + the staged residual
        // -> bf16, written back in place; no barrier among these warps (the store warp takes over)
        const int ew = warp - EPI_WARP0, half = ew >> 2;
        const int er = ((ew & 3) << 5) | lane;
        const uint32_t tlane = tmem + ((uint32_t)((ew & 3) * 32) << 16);
        const bool leader = tid == EPI_WARP0 * 32;
        int u = u0, s = have0 ? x0.s0 : 0;
        Unit x = x0;
        bool have = have0;
        int job = 0;
        while (have) {
            const int eb_i = job % NEB;
            unsigned char* eb = ebuf + eb_i * EBUF;
            const int b = job % NOB;
            const int w = min(SW, a.dv - s * SW);
            mbar_wait(r_full + eb_i, (job / NEB) & 1);
            if (job == 2 && leader) ltr(ls_sh, 12);
            mbar_wait(o_full + b, (job / NOB) & 1);
            tc_fence_after();
            if (job == 0 && leader) ltr(ls_sh, 4);
            if (job == 2 && leader) ltr(ls_sh, 13);
            constexpr int HC = SW / 2;  // columns per thread: its half of the slice
            if (half * HC < w) {
                const int c0 = half * HC;
                unsigned char* boxp = eb + (c0 >> 6) * CH;
                const int u0 = (c0 & 63) >> 3;
                // the TMEM loads and the residual reads in flight before one wait
                uint32_t o[HC];
#pragma unroll
                for (int c32 = 0; c32 < HC / 32; c32++) tmem_ld32_nw(tlane + OCOL + b * SW + c0 + c32 * 32, o + 32 * c32);
                uint4 rr[HC / 8];
#pragma unroll
                for (int k = 0; k < HC / 8; k++) rr[k] = *(const uint4*)(boxp + sw128_off(er, u0 + k));
                tmem_wait_ld();
#pragma unroll
                for (int k = 0; k < HC / 8; k++) {
                    uint32_t* h = (uint32_t*)&rr[k];
#pragma unroll
                    for (int e2 = 0; e2 < 4; e2++) {
                        const float lo = __uint_as_float(h[e2] << 16), hi = __uint_as_float(h[e2] & 0xffff0000u);
                        const __nv_bfloat162 ov =
                            __floats2bfloat162_rn(__fadd_rn(__uint_as_float(o[8 * k + 2 * e2]), lo),
                                                  __fadd_rn(__uint_as_float(o[8 * k + 2 * e2 + 1]), hi));
                        h[e2] = *(const uint32_t*)&ov;
                    }
                    *(uint4*)(boxp + sw128_off(er, u0 + k)) = rr[k];
                }
            }
            tc_fence_before();
            mbar_arrive(o_free + b);
            fence_async_smem();  // generic-proxy tile writes -> the TMA store engine
            mbar_arrive(staged + eb_i);
            if (job == 2 && leader) ltr(ls_sh, 14);
            if (leader && (job == 0 || job == 4 || job == 9)) ltr(ls_sh, job == 0 ? 5 : (job == 4 ? 6 : 7));
            if (++s >= x.s1) {
                u += gridDim.x;
                have = seek_unit(a, sc, u, x);
                s = x.s0;
            }
            job++;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    if (tid == 0) ltr(ls_sh, 10);
}

}  // namespace attn_short
}  // namespace fis

FIS_LTR_SETTER(fis_ltr_set_short)

// Would fis_attn_short_launch take this call? Every key run <= 256 keys, no pre-residual output,
// bf16 residual / output with 16-byte rows, at most MAX_RUNS runs. Batch 1 included: with slice
// groups spreading a few query tiles over the SMs it beats the general kernel's d-split / single-
// block paths there too (C2 batch-1 step 0.982 -> 0.918 ms, dense step 1.49 -> 1.42 ms).
// FIS_ATTN_SHORT=0 disables it (the general kernel's d-split / single-block modes then run).
int fis_attn_short_ok(const fis_attn_args* a) {
    // read per call (tests switch it to cover the general kernel's modes; calls run at capture time)
    const char* env = getenv("FIS_ATTN_SHORT");
    if (env && env[0] == '0') return 0;
    const int maxk = a->nseg > 0 ? a->max_seg_k : a->n_keys;
    if (maxk < 1 || maxk > 256 || a->pre.ptr || !a->res.ptr || a->res.dtype != FIS_BF16 || (a->res.ld % 8) ||
        (((uintptr_t)a->res.ptr) & 15) || a->res.step_stride || a->out.dtype != FIS_BF16 || (a->out.ld % 8) ||
        (((uintptr_t)a->out.ptr) & 15) || (a->out.step_stride % 16) || (a->dv % 64) || (a->d % 64) ||
        a->nseg > fis::attn_short::MAX_RUNS)
        return 0;
    return 1;
}

// Launches the call on the short-run kernel: FIS_OK / FIS_ERR_LAUNCH, or -1 when the call is not
// this kernel's (fis_attn's general kernel runs it).
int fis_attn_short_launch(const fis_attn_args* a, cudaStream_t stream) {
    using namespace fis::attn_short;
    if (!fis_attn_short_ok(a)) return -1;
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (nsm <= 0) nsm = 148;
    }
    const int maxk = a->nseg > 0 ? a->max_seg_k : a->n_keys;
    const int KP = (maxk + 15) / 16 * 16;
    // runs <= 128 keys: the 128-key configuration (128-column slices) on large grids; on grids of
    // < 16 query tiles (batch 1) the 256-key one, whose 64-column slices give twice the slice groups
    // (C2 batch-1 step 918 -> 903 us). FIS_ATTN_SHORT_W64: 1 forces 64-column slices, 2 forbids them
    static int w64 = getenv("FIS_ATTN_SHORT_W64") ? atoi(getenv("FIS_ATTN_SHORT_W64")) : 0;
    const bool few_tiles = (a->m + 127) / 128 < 16;
    const bool small = KP <= 128 && (w64 == 2 || (w64 == 0 && !few_tiles));
    CUtensorMap tq, tq16, tk, tv, tr, to, to8;
    if (!encode_2d(&tq, a->q.ptr, a->m, a->d, a->q.ld, 128) || !encode_2d(&tq16, a->q.ptr, a->m, a->d, a->q.ld, 16) || !encode_2d(&tk, a->k.ptr, a->n_keys, a->d, a->k.ld, KP) ||
        !encode_2d(&tv, a->vt.ptr, a->dv, a->n_keys, a->vt.ld, small ? 128 : 64) ||
        !encode_2d(&tr, a->res.ptr, a->m, a->dv, a->res.ld, 128))
        return -1;
    // output maps (whole tiles / 8-row groups); a per-step output stride takes the row-store path
    if (a->out.step_stride) {
        std::memset(&to, 0, sizeof(to));
        std::memset(&to8, 0, sizeof(to8));
    } else if (!encode_2d(&to, a->out.ptr, a->m, a->dv, a->out.ld, 128) ||
               !encode_2d(&to8, a->out.ptr, a->m, a->dv, a->out.ld, 8)) {
        return -1;
    }
    // slice groups (the kernel picks G = SMs / tiles when 0): split each query tile's value slices
    // over G units when the tiles alone leave SMs idle (each group recomputes S from L2)
    static int g_env = getenv("FIS_ATTN_SHORT_G") ? atoi(getenv("FIS_ATTN_SHORT_G")) : 0;
    static bool configured = false;
    if (!configured) {
        if (cudaFuncSetAttribute(attn_short_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<128>()) !=
                cudaSuccess ||
            cudaFuncSetAttribute(attn_short_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<256>()) !=
                cudaSuccess)
            return -1;
        configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)nsm);  // persistent: one CTA per SM loops over the units
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = small ? smem_bytes<128>() : smem_bytes<256>();
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = fis_pdl_enabled() ? 1 : 0;
    const cudaError_t e = small ? cudaLaunchKernelEx(&cfg, attn_short_kernel<128>, *a, tq, tq16, tk, tv, tr, to, to8, KP, g_env)
                                    : cudaLaunchKernelEx(&cfg, attn_short_kernel<256>, *a, tq, tq16, tk, tv, tr, to, to8, KP, g_env);
    return e == cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
}
