// Fused attention on tcgen05 with TMA operand staging (sm_100a).
//
//   out[r, c0:c0+dvs] = res + softmax(Q K^T * scale) (V^T)^T      (unet.py:279-293, sparse.py:265-361)
//
// One CTA = one 128-query tile x one value slice (dvs <= 256 columns) of one segment. Ragged
// segments (batched requests) restrict each query run to its own key run.
//
//   warp 4 (lane 0) : TMA producer. Per 64-wide chunk: Q {64 x 128} + K {64 x 128} for a score
//                     block, or V^T {64 keys x dvs} for a P.V block; one expect_tx per stage.
//                     Rows past the end of a matrix are zero-filled by TMA; rows of a neighbouring
//                     segment are masked in the softmax (P = 0).
//   warp 5          : TMEM allocator + MMA issuer: S_j = Q K_j^T into one of two 128-column TMEM
//                     buffers, O += P_j V_j into 256 columns; pass 2 issues S_{j+1} before P_j.V_j so
//                     the tensor core works while the softmax warps read S_j.
//   warps 0-3       : softmax (thread = query row): pass 1 keeps the running max / sum over all
//                     key blocks, pass 2 writes P_j = exp(s - m) / l as bf16 into one of two SW128
//                     P tiles; then the epilogue (O + residual -> out).
// A segment of <= 128 keys takes one pass (statistics and P from the same S).
#include "fis_attn.cuh"
#include "fis_tma.cuh"
#include <cstring>

namespace fis {
namespace attn {

using namespace fis::tc;

constexpr int THREADS = 192, TMA_WARP = 4, MMA_WARP = 5;
// a stage holds a Q chunk + a K chunk (S block) or one V^T chunk (<= 256 rows x 64 keys): 32 KB,
// four of them (128 KB of operands in flight per CTA; the S passes are bound by bytes in flight)
constexpr int STAGES = 4;
constexpr int A_BYTES = 128 * 64 * 2;            // Q chunk (K chunk at +A_BYTES)
constexpr int STAGE = 2 * A_BYTES;               // = V^T chunk bytes at dvs = 256
constexpr int P_BYTES = 2 * 128 * 64 * 2;        // P tile: 128 rows x 128 keys, two 64-key SW128 chunks
// d-split receive buffer (P_DSPLIT: peers' fp32 partial-S row slices), starting at P tile 1
constexpr int RX_EXTRA = 24 * 1024;
constexpr int SMEM = STAGES * STAGE + 2 * P_BYTES + RX_EXTRA + 1024 + 256 + 1024;  // + key-split statistics exchange
constexpr uint32_t O_COL = 256;                  // TMEM: S buffers at 0 / 128, O at 256
constexpr int EPI_LD = 256 + 4;                  // O staging row pitch (floats; spans the stages + P tiles)
// P sharing across the value slices of a query tile (segments of <= 256 keys): a P_OUT launch
// (slice 0 only) computes S, the softmax and writes P (bf16, [row][256]) to scratch; the P_IN
// launch (every slice) TMA-loads those P tiles and runs only P.V + the epilogue
// P_OUT_KS: P_OUT for two-block key runs split over a 2-CTA cluster (CTA = one key block); the
// row max / sum of the two blocks are exchanged through distributed shared memory
// P_DSPLIT (batch 1, <= 128 keys): the value-slice CTAs of a query tile form a cluster and split the
// S reduction (the head dim d) between them instead of each recomputing all of S: CTA z computes
// the partial S over its d chunks, pushes the partial row slices to their owners (DSMEM bulk
// copies), owners sum the partials in cluster-rank order, run the softmax of their rows and push
// the bf16 P rows into every CTA's P tile; each CTA then runs P.V for its value slice.
constexpr int P_NONE = 0, P_OUT = 1, P_IN = 2, P_OUT_KS = 3, P_DSPLIT = 4;
// flag on P_NONE: runs of >= 3 key blocks take ONE pass (online softmax: P_j = 2^(s - m_run) with a
// lazily raised running max, O rescaled in TMEM only when a block's max exceeds m_run by > 8, O / l
// in the epilogue) instead of a statistics pass that recomputes every S block
constexpr int P_ONEPASS_OK = 8;
// flag on P_NONE (batch 1, no segments): the key run is split over gridDim.z CTAs per (query tile,
// value slice) -- flash-decoding style: each runs the one-pass loop over its key blocks and writes
// its unnormalised O rows + (running max, sum) to the workspace; after a group barrier (arrive /
// depart counters; the grid is below one wave) every split CTA merges 128 / splits rows of the
// tile in split order (deterministic), adds the residual and stores
constexpr int P_SPLITKV = 16;
// flag: the epilogue TMA-loads the residual tile (32-column SW64 boxes) into the P tiles, adds O in
// place and TMA-stores whole 8-row groups (host-encoded maps tr / to / to8) instead of staging O in
// fp32 and storing 16-byte runs with LDG residual loads (7-10 us of a batch-1 d = 1280 call)
constexpr int P_FEPI = 32;
constexpr float RESCALE_SLACK = 8.f;  // log2 units: unnormalised P <= 2^8

// The MMA order (and so the producer's load order) of one pass: S blocks 0..nkb-1; in pass 2
// step u issues S_u (u < nkb) and then P_{u-1}.V_{u-1} (u >= 1).
__global__ void __launch_bounds__(THREADS, 1)
    attn_kernel(const fis_attn_args a, const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tp,
                const __grid_constant__ CUtensorMap tr, const __grid_constant__ CUtensorMap to,
                const __grid_constant__ CUtensorMap to8, int dvs, int pmode_in) {
    const bool onepass_ok = (pmode_in & P_ONEPASS_OK) != 0;
    const bool splitkv = (pmode_in & P_SPLITKV) != 0;
    const bool fepi = (pmode_in & P_FEPI) != 0 && !splitkv;
    pmode_in &= ~(P_ONEPASS_OK | P_SPLITKV | P_FEPI);
    const bool ks = pmode_in == P_OUT_KS;
    const bool dsp = pmode_in == P_DSPLIT;
    const int pmode = ks ? P_OUT : (dsp ? P_NONE : pmode_in);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* ptile = smem + STAGES * STAGE;
    float* rxbuf = (float*)(ptile + P_BYTES);  // P_DSPLIT receive slots (P tile 1 + RX_EXTRA)
    uint64_t* full = (uint64_t*)(ptile + 2 * P_BYTES + RX_EXTRA);
    uint64_t* empty = full + STAGES;
    uint64_t* s_ready = empty + STAGES;  // [2]
    uint64_t* s_free = s_ready + 2;      // [2]
    uint64_t* p_ready = s_free + 2;      // [2]
    uint64_t* p_free = p_ready + 2;      // [2]
    uint64_t* o_done = p_free + 2;
    uint64_t* rx_bar = o_done + 1;       // P_DSPLIT: peers' partial row slices landed (one phase per round)
    uint64_t* tx_ok = rx_bar + 1;        // P_DSPLIT: every peer consumed its receive buffer (per round)
    uint64_t* part_free = tx_ok + 1;     // P_DSPLIT, 2 key blocks: stages 2-3 free for V^T of block 1
    uint64_t* res_bar = part_free + 1;   // P_FEPI: the residual tile landed
    uint32_t* tmem_slot = (uint32_t*)(res_bar + 1);
    float2* xst = (float2*)(ptile + 2 * P_BYTES + RX_EXTRA + 256);  // [128] key-split (max, sum) exchange

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ls = ltr_begin(2 + pmode_in * 16);  // thread 0 of CTA (0,0,0) only
    int q_beg = 0, q_end = a.m, k_beg = 0, n_keys = a.n_keys;
    if (a.nseg > 0) {
        const int sg = blockIdx.z;
        q_beg = __ldg(a.q_seg + 2 * sg);
        q_end = __ldg(a.q_seg + 2 * sg + 1);
        k_beg = __ldg(a.k_seg + 2 * sg);
        n_keys = __ldg(a.k_seg + 2 * sg + 1) - k_beg;
    }
    const int m0 = q_beg + blockIdx.y * 128, c0 = ks ? 0 : blockIdx.x * dvs;
    if (m0 >= q_end || n_keys <= 0) return;  // uniform for the CTA (and its cluster peer), before any barrier
    // key split: this CTA owns key block blockIdx.x of the run; a run of <= 128 keys leaves CTA 1 idle
    const int kb_off = ks ? (int)blockIdx.x * 128 : 0;
    bool idle = false;
    if (ks) {
        k_beg += kb_off;
        n_keys -= kb_off;
        if (n_keys <= 0) {
            idle = true;
            n_keys = 1;
        }
        if (n_keys > 128) n_keys = 128;
    }
    // split-KV: this CTA's key blocks [kv0, kv0 + kvper) of the run
    const int kvs = splitkv ? (int)gridDim.z : 1, kvz = splitkv ? (int)blockIdx.z : 0;
    const int kvper = splitkv ? ((n_keys + 127) / 128 + kvs - 1) / kvs : 0;
    if (splitkv) {
        k_beg += kvz * kvper * 128;
        n_keys = min(n_keys - kvz * kvper * 128, kvper * 128);  // >= 1 (host: every split owns a block)
    }
    const int nkb = (n_keys + 127) / 128, dch = a.d / 64;
    const bool single = nkb == 1 && !splitkv;
    // two key blocks: both S blocks stay resident in the two TMEM buffers, so the statistics pass
    // and the P pass read the same S (no recompute, half the Q/K traffic)
    const bool resident = nkb == 2 && !splitkv;
    const bool onepass = (onepass_ok && pmode == P_NONE && !dsp && nkb >= 3) || splitkv;
    const int first_pass = (single || onepass) ? 2 : 1;
    const int pw = ((a.max_seg_k + 127) / 128) * 128;  // P scratch row width (P sharing)
    // P_DSPLIT: cluster rank = value slice; this CTA's d chunks [kc0, kc1) and owned rows [rbeg, rend)
    const int cs = dsp ? (int)gridDim.x : 1, rank = (int)blockIdx.x;
    const int kc0 = dsp ? rank * dch / cs : 0, kc1 = dsp ? (rank + 1) * dch / cs : dch;
    const int rp = (128 + cs - 1) / cs;
    const int rbeg = min(128, rank * rp), rend = min(128, rbeg + rp);
    if (tid == 0) {
        for (int i = 0; i < STAGES; i++) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(s_ready + b, 1);
            mbar_init(s_free + b, 128);
            mbar_init(p_ready + b, (pmode == P_IN || dsp) ? 1 : 128);
            mbar_init(p_free + b, 1);
        }
        mbar_init(o_done, 1);
        mbar_init(rx_bar, 1);
        mbar_init(tx_ok, cs > 1 ? cs - 1 : 1);
        mbar_init(part_free, 1);
        mbar_init(res_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (dsp && rend > rbeg)  // incoming: cs - 1 partial slices of this CTA's rows
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(rx_bar)),
                         "r"((uint32_t)((cs - 1) * (rend - rbeg) * 512))
                         : "memory");
    }
    if (warp == TMA_WARP && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tq) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tk) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tv) : "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (dsp) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");  // barriers initialised
    const int t = cur_step(a.step);  // host-written before the step: safe to read before the wait
    ltr(ls, 1);
    if (warp == TMA_WARP && lane == 0 && a.nseg == 0 && !idle) {
        // cross attention: K and V^T are the per-edit text keys / values (no kernel of the step writes
        // them) -> pull this CTA's chunks into L2 while the previous kernel runs. Self attention reads
        // K / V from the QKV GEMM just before it (already in L2): K lives in the Q buffer's rows.
        // self attention passes the keys as the layer input s (written by the kernel before the
        // projection): only the cross-attention text matrices are prefetched (K with a different
        // row count than the queries, or V^T narrower than the query count)
        const bool self_kv = a.n_keys == a.m;
        if (!self_kv) {
            const int nkb2 = (n_keys + 127) / 128;
            for (int j = 0; j < nkb2; j++)
                for (int kc = kc0; kc < kc1; kc++) tma_prefetch2d(&tk, kc * 64, k_beg + j * 128);
            for (int j = 0; j < nkb2; j++)
                for (int h = 0; h < 2; h++) tma_prefetch2d(&tv, k_beg + j * 128 + h * 64, c0);
        }
    }
    pdl_trigger();
    pdl_wait();
    ltr(ls, 2);

    if (idle && warp != TMA_WARP && warp != MMA_WARP) goto ks_softmax;
    if (idle) goto done;
    if (ks && warp < 4) goto ks_softmax;
    if (warp == TMA_WARP) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            const uint32_t sbase = smem_u32(smem);
            int it = 0;
            auto stage = [&](uint32_t bytes) {
                const int st = it % STAGES;
                if (it >= STAGES) mbar_wait(empty + st, ((it / STAGES) & 1) ^ 1);
                arrive_expect_tx(full + st, bytes);
                it++;
                return st;
            };
            auto load_s = [&](int j) {
                for (int kc = 0; kc < dch; kc++) {
                    const int st = stage(2 * A_BYTES);
                    const uint32_t sa = sbase + st * STAGE;
                    tma2d(sa, &tq, kc * 64, m0, full + st);
                    tma2d(sa + A_BYTES, &tk, kc * 64, k_beg + j * 128, full + st);
                }
            };
            auto load_v = [&](int j) {
                for (int h = 0; h < 2; h++) {
                    const int st = stage((uint32_t)(dvs * 64 * 2));
                    tma2d(sbase + st * STAGE, &tv, k_beg + j * 128 + h * 64, c0, full + st);
                }
            };
            if (dsp) {
                // this CTA's d chunks of every S block, the ring padded to a whole cycle (empty
                // stages complete at once), then V^T of block 0 into stages 0-1 (the partial-S
                // exchange buffer lives in stages 2-3) and, once the exchange is over, block 1's
                for (int kc = kc0; kc < kc1; kc++)
                    for (int j = 0; j < nkb; j++) {
                        const int st = stage(2 * A_BYTES);
                        const uint32_t sa = sbase + st * STAGE;
                        tma2d(sa, &tq, kc * 64, m0, full + st);
                        tma2d(sa + A_BYTES, &tk, kc * 64, k_beg + j * 128, full + st);
                    }
                while (it % STAGES) stage(0);
                load_v(0);
                if (nkb > 1) {
                    mbar_wait(part_free, 0);
                    load_v(1);
                }
            } else if (pmode == P_IN) {  // P tiles of this query tile from the scratch (written by the P_OUT launch)
                for (int j = 0; j < nkb; j++) {
                    const int pb = j & 1;
                    if (j >= 2) mbar_wait(p_free + pb, ((j >> 1) & 1) ^ 1);  // P.V_{j-2} done with the buffer
                    arrive_expect_tx(p_ready + pb, (uint32_t)P_BYTES);
                    for (int h = 0; h < 2; h++)
                        tma2d(smem_u32(ptile) + pb * P_BYTES + h * (128 * 128), &tp, j * 128 + h * 64, m0,
                              p_ready + pb);
                    load_v(j);
                }
            } else if (pmode == P_OUT) {  // statistics pass (unless S is resident) + P pass
                if (!(resident || single))
                    for (int j = 0; j < nkb; j++) load_s(j);
                for (int j = 0; j < nkb; j++) load_s(j);
            } else if (resident) {
                load_s(0);
                load_s(1);
                load_v(0);
                load_v(1);
            } else {
                if (!single && !onepass)
                    for (int j = 0; j < nkb; j++) load_s(j);
                for (int u = 0; u <= nkb; u++) {
                    if (u < nkb) load_s(u);
                    if (u >= 1) load_v(u - 1);
                }
            }
        }
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t sbase = smem_u32(smem), pbase = smem_u32(ptile);
        const uint32_t id_s = idesc_bf16(128, 128), id_o = idesc_bf16(128, dvs);
        int it = 0, sb = 0;
        auto mma_s = [&]() {
            const int b = sb & 1;
            if (sb >= 2) mbar_wait(s_free + b, ((sb >> 1) & 1) ^ 1);  // softmax has read S_{sb-2}
            for (int kc = 0; kc < dch; kc++) {
                const int st = it % STAGES;
                mbar_wait(full + st, (it / STAGES) & 1);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t sa = sbase + st * STAGE, sbb = sa + A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < 4; kk++)
                        mma_bf16(tmem + b * 128, sw128_desc(sa + kk * 32), sw128_desc(sbb + kk * 32), id_s,
                                 (kc | kk) ? 1u : 0u);
                    mma_commit(empty + st);
                    if (kc == dch - 1) mma_commit(s_ready + b);
                }
                __syncwarp();
                it++;
            }
            sb++;
        };
        auto mma_pv = [&](int j) {
            const int pb = j & 1;
            mbar_wait(p_ready + pb, (j >> 1) & 1);  // P_j written
            for (int h = 0; h < 2; h++) {
                const int st = it % STAGES;
                mbar_wait(full + st, (it / STAGES) & 1);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t sbb = sbase + st * STAGE;  // V^T chunk
                    const uint32_t pa = pbase + pb * P_BYTES + h * (128 * 128);
#pragma unroll
                    for (int kk = 0; kk < 4; kk++)
                        mma_bf16(tmem + O_COL, sw128_desc(pa + kk * 32), sw128_desc(sbb + kk * 32), id_o,
                                 (j | h | kk) ? 1u : 0u);
                    mma_commit(empty + st);
                    if (h == 1) {
                        mma_commit(p_free + pb);
                        if (j == nkb - 1) mma_commit(o_done);
                    }
                }
                __syncwarp();
                it++;
            }
        };
        if (dsp) {
            for (int kc = kc0; kc < kc1; kc++)
                for (int j = 0; j < nkb; j++) {
                    const int st = it % STAGES;
                    mbar_wait(full + st, (it / STAGES) & 1);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t sa = sbase + st * STAGE, sbb = sa + A_BYTES;
#pragma unroll
                        for (int kk = 0; kk < 4; kk++)
                            mma_bf16(tmem + j * 128, sw128_desc(sa + kk * 32), sw128_desc(sbb + kk * 32), id_s,
                                     (kc != kc0 || kk) ? 1u : 0u);
                        mma_commit(empty + st);
                        if (kc == kc1 - 1) mma_commit(s_ready + j);
                    }
                    __syncwarp();
                    it++;
                }
            while (it % STAGES) {  // the producer's padding stages
                const int st = it % STAGES;
                mbar_wait(full + st, (it / STAGES) & 1);
                if (lane == 0) mma_commit(empty + st);
                __syncwarp();
                it++;
            }
            for (int j = 0; j < nkb; j++) mma_pv(j);
        } else if (pmode == P_IN) {
            for (int j = 0; j < nkb; j++) mma_pv(j);
        } else if (pmode == P_OUT) {
            if (!(resident || single))
                for (int j = 0; j < nkb; j++) mma_s();
            for (int j = 0; j < nkb; j++) mma_s();
        } else if (resident) {
            mma_s();
            mma_s();
            mma_pv(0);
            mma_pv(1);
        } else {
            if (!single && !onepass)
                for (int j = 0; j < nkb; j++) mma_s();
            for (int u = 0; u <= nkb; u++) {
                if (u < nkb) mma_s();
                if (u >= 1) mma_pv(u - 1);
            }
        }
    } else {
        // ------------------------------------------------------------ softmax + epilogue (warps 0-3)
        const int lr = tid, r = m0 + lr;
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        // softmax in the log2 domain: x = s * scale * log2(e); P = 2^(x - m - log2 l) (one FFMA + EX2)
        const float sl = a.scale * 1.4426950408889634f;
        float mrow = -INFINITY, lrow = 0.f;
        int sb = 0;
        float v[32];
        if (dsp) {
            // per key block j (round j): 1. the partial S_j (this CTA's d chunks) -> part: fp32
            // [128][128] in stages 2-3, 16-byte units XOR-swizzled by row (conflict-free row-per-
            // thread writes; rows stay contiguous); 2. each peer's row slice -> its receive slot for
            // this rank (DSMEM bulk copy); 3. the owned rows' partials summed in rank order. Then the
            // softmax of the owned rows over all blocks and the bf16 P rows -> every CTA's P tiles.
            // 4 threads per owned row (32 keys of each block); two row iterations when a CTA owns 64
            // rows (one key block only)
            unsigned char* part = smem + 2 * STAGE;
            const uint32_t part_s = smem_u32(part);
            const int own = rend - rbeg;
            const int seg = tid & 3, kbase = seg * 32;
            const int niter = (own + 31) >> 5;
            float xs[2][32];
            auto sum_rows = [&](float (&x)[32], int i) {
                const int r = rbeg + i;
#pragma unroll
                for (int q = 0; q < 32; q++) x[q] = 0.f;
                if (i >= own) return;
                for (int z = 0; z < cs; z++) {
                    const unsigned char* src = z == rank ? part + r * 512
                                                         : (const unsigned char*)rxbuf + (z < rank ? z : z - 1) * rp * 512 + i * 512;
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const int u = seg * 8 + q;
                        const float4 f = *(const float4*)(src + ((u ^ (r & 7)) << 4));
                        x[4 * q] += f.x; x[4 * q + 1] += f.y; x[4 * q + 2] += f.z; x[4 * q + 3] += f.w;
                    }
                }
            };
            for (int j = 0; j < nkb; j++) {
                // part lives in stages 2-3: round 0 waits for EVERY S block (the last blocks' MMAs read
                // those stages after block 0 completes)
                if (j == 0)
                    for (int b = 0; b < nkb; b++) mbar_wait(s_ready + b, 0);
                if (j == 0) ltr(ls, 3);
                tc_fence_after();
                if (j > 0) asm volatile("bar.sync 3, 128;" ::: "memory");  // round j-1's copies have read part
#pragma unroll 1
                for (int cb = 0; cb < 128; cb += 32) {
                    tmem_ld32(tmem + lane_off + j * 128 + cb, v);
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const int u = (cb >> 2) + q;
                        *(float4*)(part + lr * 512 + ((u ^ (lr & 7)) << 4)) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    }
                }
                fence_async_smem();
                if (j == 0) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // peers' barriers initialised
                asm volatile("bar.sync 3, 128;" ::: "memory");
                if (tid == 0) {
                    if (j > 0) mbar_wait_cluster(tx_ok, (j - 1) & 1);  // every peer consumed round j-1
                    for (int p = 0; p < cs; p++) {
                        if (p == rank) continue;
                        const int pb = min(128, p * rp), pe = min(128, pb + rp);
                        if (pe <= pb) continue;
                        const int slot = rank < p ? rank : rank - 1;
                        uint32_t dst, bar;
                        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(smem_u32(rxbuf) + (uint32_t)(slot * rp * 512)), "r"(p));
                        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar) : "r"(smem_u32(rx_bar)), "r"(p));
                        asm volatile(
                            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                            "r"(part_s + (uint32_t)(pb * 512)), "r"((uint32_t)((pe - pb) * 512)), "r"(bar)
                            : "memory");
                    }
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                if (j == 1) ltr(ls, 9);
                if (own > 0) mbar_wait(rx_bar, j & 1);
                if (j == 0) ltr(ls, 5);
                if (j == 1) ltr(ls, 10);
                if (nkb > 1) {
                    if (j == 0) sum_rows(xs[0], tid >> 2);
                    else sum_rows(xs[1], tid >> 2);
                } else {
                    sum_rows(xs[0], tid >> 2);
                    if (niter > 1) sum_rows(xs[1], (tid >> 2) + 32);
                }
                asm volatile("bar.sync 3, 128;" ::: "memory");  // receive buffer and part fully read
                if (tid == 0) {
                    if (j + 1 < nkb && own > 0)  // re-arm for round j+1 before releasing the peers
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(rx_bar)),
                                     "r"((uint32_t)((cs - 1) * own * 512))
                                     : "memory");
                    for (int p = 0; p < cs; p++) {
                        if (p == rank) continue;
                        uint32_t rb;
                        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(tx_ok)), "r"(p));
                        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
                    }
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // round j's copies have read part
                    if (j == nkb - 1 && nkb > 1) mbar_arrive(part_free);  // V^T of block 1 may overwrite stages 2-3
                    if (j == 0) ltr(ls, 8);
                }
            }
            // softmax of one owned row (this thread's 32 keys of each block) -> the local P tiles
            auto emit = [&](const float (&x0)[32], const float (&x1)[32], int nb, int i) {
                const bool act = i < own;
                const int r = rbeg + i;
                const int lim0 = n_keys - kbase, lim1 = n_keys - 128 - kbase;
                float cm = -INFINITY;
#pragma unroll
                for (int q = 0; q < 32; q++)
                    if (q < lim0) cm = fmaxf(cm, x0[q]);
                if (nb > 1) {
#pragma unroll
                    for (int q = 0; q < 32; q++)
                        if (q < lim1) cm = fmaxf(cm, x1[q]);
                }
                cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 1));
                cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 2));
                const float mn = cm * sl;
                float add = 0.f;
#pragma unroll
                for (int q = 0; q < 32; q++)
                    if (q < lim0) add += ex2(fmaf(x0[q], sl, -mn));
                if (nb > 1) {
#pragma unroll
                    for (int q = 0; q < 32; q++)
                        if (q < lim1) add += ex2(fmaf(x1[q], sl, -mn));
                }
                add += __shfl_xor_sync(0xffffffffu, add, 1);
                add += __shfl_xor_sync(0xffffffffu, add, 2);
                const float off = mn + __log2f(add);
                if (!act) return;
                for (int b = 0; b < nb; b++) {
                    const int lim = b ? lim1 : lim0;
                    unsigned char* pt = ptile + b * P_BYTES + (kbase >> 6) * (128 * 128);
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        uint4 pk;
                        __nv_bfloat162* h = (__nv_bfloat162*)&pk;
#pragma unroll
                        for (int e2 = 0; e2 < 4; e2++) {
                            const int q0 = 8 * u + 2 * e2;
                            const float y0 = b ? x1[q0] : x0[q0], y1 = b ? x1[q0 + 1] : x0[q0 + 1];
                            const float p0 = q0 < lim ? ex2(fmaf(y0, sl, -off)) : 0.f;
                            const float p1 = q0 + 1 < lim ? ex2(fmaf(y1, sl, -off)) : 0.f;
                            h[e2] = __floats2bfloat162_rn(p0, p1);
                        }
                        *(uint4*)(pt + sw128_off(r, ((kbase & 63) >> 3) + u)) = pk;
                    }
                }
            };
            if (nkb > 1) {
                emit(xs[0], xs[1], 2, tid >> 2);
                ltr(ls, 11);
            } else {
                emit(xs[0], xs[0], 1, tid >> 2);
                if (niter > 1) emit(xs[1], xs[1], 1, (tid >> 2) + 32);
            }
            fence_async_smem();
            asm volatile("bar.sync 3, 128;" ::: "memory");
            if (tid == 0) {  // 4. the owned P rows -> every peer's P tiles; then expect the peers' rows
                // P tile 1 aliases the receive buffers: every peer has consumed its last round
                if (nkb > 1) mbar_wait_cluster(tx_ok, (nkb - 1) & 1);
                const uint32_t pt_s = smem_u32(ptile);
                if (own > 0)
                    for (int p = 0; p < cs; p++) {
                        if (p == rank) continue;
                        for (int b = 0; b < nkb; b++) {
                            uint32_t bar;
                            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar) : "r"(smem_u32(p_ready + b)), "r"(p));
                            for (int h = 0; h < 2; h++) {
                                const uint32_t off = pt_s + (uint32_t)(b * P_BYTES + h * 128 * 128 + rbeg * 128);
                                uint32_t dst;
                                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(off), "r"(p));
                                asm volatile(
                                    "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                                    "r"(off), "r"((uint32_t)(own * 128)), "r"(bar)
                                    : "memory");
                            }
                        }
                    }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                for (int b = 0; b < nkb; b++)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(p_ready + b)),
                                 "r"((uint32_t)((128 - own) * 256))
                                 : "memory");
                ltr(ls, 6);
                // the outgoing copies have read part / P before the epilogue reuses the stages
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
        }
        for (int pass = first_pass; pass <= 2 && pmode != P_IN && !dsp; pass++) {
            if (resident) sb = 0;  // pass 2 re-reads the resident S blocks (their phases already completed)
            for (int j = 0; j < nkb; j++) {
                const int b = sb & 1;
                mbar_wait(s_ready + b, (sb >> 1) & 1);
                if (sb == 0) ltr(ls, 3);
                tc_fence_after();
                const uint32_t trow = tmem + lane_off + b * 128;
                const int kbase = j * 128;
                if (pass == 1 || single) {  // row statistics (online over this block)
#pragma unroll 1
                    for (int cb = 0; cb < 128; cb += 32) {
                        tmem_ld32(trow + cb, v);
                        const int lim = n_keys - kbase - cb;  // valid keys in this chunk
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
                }
                if (pass == 2 && pmode == P_OUT) {  // P_j -> the P scratch row (keys of this segment)
                    const float off = mrow + __log2f(lrow);
                    __nv_bfloat16* prow = (__nv_bfloat16*)a.ws + (long long)r * pw + kbase;
#pragma unroll 1
                    for (int cb = 0; cb < 128; cb += 32) {
                        tmem_ld32(trow + cb, v);
                        const int lim = n_keys - kbase - cb;
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            uint4 pk;
                            __nv_bfloat162* h = (__nv_bfloat162*)&pk;
#pragma unroll
                            for (int e2 = 0; e2 < 4; e2++) {
                                const int q0 = 8 * u + 2 * e2;
                                const float p0 = q0 < lim ? ex2(fmaf(v[q0], sl, -off)) : 0.f;
                                const float p1 = q0 + 1 < lim ? ex2(fmaf(v[q0 + 1], sl, -off)) : 0.f;
                                h[e2] = __floats2bfloat162_rn(p0, p1);
                            }
                            if (r < q_end) *(uint4*)(prow + cb + 8 * u) = pk;
                        }
                    }
                    tc_fence_before();
                    if (!resident) mbar_arrive(s_free + b);
                } else if (pass == 2) {  // P_j -> bf16 P tile j & 1 (SW128, K-major)
                    const int pb = j & 1;
                    float off;
                    if (onepass) {
                        float cm = -INFINITY;
#pragma unroll 1
                        for (int cb = 0; cb < 128; cb += 32) {
                            tmem_ld32(trow + cb, v);
                            const int lim = n_keys - kbase - cb;
#pragma unroll
                            for (int q = 0; q < 32; q++)
                                if (q < lim) cm = fmaxf(cm, v[q]);
                        }
                        const float mb = cm * sl;
                        if (j == 0) mrow = mb;
                        const bool need = j > 0 && mb > mrow + RESCALE_SLACK;
                        if (__any_sync(0xffffffffu, need)) {  // warp-collective TMEM access
                            mbar_wait(p_free + ((j - 1) & 1), ((j - 1) >> 1) & 1);  // P.V_{j-1} done: O stable
                            tc_fence_after();
                            const float f = need ? ex2(mrow - mb) : 1.f;
#pragma unroll 1
                            for (int cb = 0; cb < dvs; cb += 32) {
                                tmem_ld32(tmem + lane_off + O_COL + cb, v);
#pragma unroll
                                for (int q = 0; q < 32; q++) v[q] *= f;
                                tmem_st32(tmem + lane_off + O_COL + cb, v);
                            }
                            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                            if (need) {
                                lrow *= f;
                                mrow = mb;
                            }
                        }
                        off = mrow;
                    } else {
                        off = mrow + __log2f(lrow);
                    }
                    if (j >= 2) mbar_wait(p_free + pb, ((j >> 1) & 1) ^ 1);  // P.V_{j-2} done
                    unsigned char* pt0 = ptile + pb * P_BYTES;
                    float psum = 0.f;
#pragma unroll 1
                    for (int cb = 0; cb < 128; cb += 32) {
                        tmem_ld32(trow + cb, v);
                        const int lim = n_keys - kbase - cb;
                        unsigned char* pt = pt0 + (cb >> 6) * (128 * 128);
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            uint4 pk;
                            __nv_bfloat162* h = (__nv_bfloat162*)&pk;
#pragma unroll
                            for (int e2 = 0; e2 < 4; e2++) {
                                const int q0 = 8 * u + 2 * e2;
                                const float p0 = q0 < lim ? ex2(fmaf(v[q0], sl, -off)) : 0.f;
                                const float p1 = q0 + 1 < lim ? ex2(fmaf(v[q0 + 1], sl, -off)) : 0.f;
                                psum += p0 + p1;
                                h[e2] = __floats2bfloat162_rn(p0, p1);
                            }
                            const int unit = ((cb & 63) >> 3) + u;
                            *(uint4*)(pt + sw128_off(lr, unit)) = pk;
                        }
                    }
                    if (onepass) lrow += psum;
                    tc_fence_before();
                    // S_j fully read (resident S blocks are never re-issued: nobody waits on s_free, and
                    // a second arrival per thread without a wait in between is a barrier misuse)
                    if (!resident) mbar_arrive(s_free + b);
                    fence_async_smem();       // generic-proxy P writes -> tensor-core reads
                    mbar_arrive(p_ready + pb);
                } else {
                    tc_fence_before();
                    if (!resident) mbar_arrive(s_free + b);
                }
                sb++;
            }
        }
        // epilogue: stage the O row slice (fp32) in the idle pipeline stages; the stores run below
        if (pmode == P_OUT) goto done;
        mbar_wait(o_done, 0);
        if (splitkv) {
            // partial rows [tile][slice][split][128][dvs + 4] (O unnormalised, then max, sum; 16-B rows)
            tc_fence_after();
            const int nsl = a.dv / dvs, grp = blockIdx.y * nsl + blockIdx.x;
            const int pitch = dvs + 4;
            float* pbase = (float*)a.ws + (long long)grp * kvs * 128 * pitch;
            float* mine = pbase + ((long long)kvz * 128 + lr) * pitch;
#pragma unroll 1
            for (int cb = 0; cb < dvs; cb += 32) {
                tmem_ld32(tmem + lane_off + O_COL + cb, v);
#pragma unroll
                for (int q = 0; q < 8; q++)
                    __stcg((float4*)(mine + cb + 4 * q), make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
            }
            __stcg(mine + dvs, mrow);
            __stcg(mine + dvs + 1, lrow);
            __threadfence();
            asm volatile("bar.sync 3, 128;" ::: "memory");
            // every split CTA of the group waits for all partials (the groups' CTAs are co-resident:
            // the grid is below one wave), then merges its own 128 / kvs rows
            int* arrive = (int*)((char*)a.ws + a.ws_bytes) - 1024 + 2 * grp;
            int* depart = arrive + 1;
            if (tid == 0) {
                atomicAdd(arrive, 1);
                int seen;
                do {
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(seen) : "l"(arrive) : "memory");
                } while (seen < kvs);
            }
            asm volatile("bar.sync 3, 128;" ::: "memory");
            __threadfence();
            // per-row merge weights: w_z = 2^(m_z - M) / sum_z l_z 2^(m_z - M)
            __shared__ float sw[128][8];
            const int rpc = (128 + kvs - 1) / kvs, rb0 = min(128, kvz * rpc), rb1 = min(128, rb0 + rpc);
            if (lr >= rb0 && lr < rb1) {
                float mz[8];
                float M = -INFINITY;
                for (int z = 0; z < kvs; z++) {
                    mz[z] = __ldcg(pbase + ((long long)z * 128 + lr) * pitch + dvs);
                    M = fmaxf(M, mz[z]);
                }
                float Ls = 0.f;
                for (int z = 0; z < kvs; z++)
                    Ls = fmaf(__ldcg(pbase + ((long long)z * 128 + lr) * pitch + dvs + 1), ex2(mz[z] - M), Ls);
                const float inv = 1.f / Ls;
                for (int z = 0; z < kvs; z++) sw[lr][z] = ex2(mz[z] - M) * inv;
            }
            asm volatile("bar.sync 3, 128;" ::: "memory");
            char* ob = ref_base(a.out, t);
            char* pbp = a.pre.ptr ? ref_base(a.pre, t) : nullptr;
            const char* rb = a.res.ptr ? ref_base(a.res, t) : nullptr;
            const int chunks = dvs / 16, nrows = max(0, min(rb1, q_end - m0) - rb0), total = nrows * chunks;
            // items (row, 16-column chunk), consecutive threads on consecutive chunks of a row;
            // 2 items per thread in flight (their partial-chunk loads issued before use)
#pragma unroll 1
            for (int i0 = tid; i0 < total; i0 += 256) {
                float w[2][16], q[2][16];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int item = i0 + 128 * h;
#pragma unroll
                    for (int e2 = 0; e2 < 16; e2++) w[h][e2] = 0.f;
                    if (item >= total) continue;
                    const int rr = rb0 + item / chunks, cb = (item % chunks) * 16;
                    if (rb) load_row16(rb, a.res.dtype, (long long)(m0 + rr) * a.res.ld + c0 + cb, 16, q[h]);
                    for (int z = 0; z < kvs; z++) {
                        const float* src = pbase + ((long long)z * 128 + rr) * pitch + cb;
                        const float wt = sw[rr][z];
#pragma unroll
                        for (int e4 = 0; e4 < 4; e4++) {
                            const float4 f = __ldcg((const float4*)(src + 4 * e4));
                            w[h][4 * e4] = fmaf(f.x, wt, w[h][4 * e4]);
                            w[h][4 * e4 + 1] = fmaf(f.y, wt, w[h][4 * e4 + 1]);
                            w[h][4 * e4 + 2] = fmaf(f.z, wt, w[h][4 * e4 + 2]);
                            w[h][4 * e4 + 3] = fmaf(f.w, wt, w[h][4 * e4 + 3]);
                        }
                    }
                }
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int item = i0 + 128 * h;
                    if (item >= total) continue;
                    const int rr = rb0 + item / chunks, cb = (item % chunks) * 16;
                    const long long row = m0 + rr;
                    if (pbp) store_row16(pbp, a.pre.dtype, row * a.pre.ld + c0 + cb, 16, w[h]);
                    if (rb) {
#pragma unroll
                        for (int e2 = 0; e2 < 16; e2++) w[h][e2] = __fadd_rn(w[h][e2], q[h][e2]);
                    }
                    store_row16(ob, a.out.dtype, row * a.out.ld + c0 + cb, 16, w[h]);
                }
            }
            if (tid == 0 && atomicAdd(depart, 1) == kvs - 1) {  // everyone is past the wait: reset
                *arrive = 0;
                *depart = 0;
            }
            goto done;
        }
        ltr(ls, 4);
        tc_fence_after();
        if (dsp) asm volatile("bar.sync 3, 128;" ::: "memory");  // thread 0's outgoing copies done reading
        const float inv_l = onepass ? 1.f / lrow : 1.f;  // one pass: O holds the unnormalised sum
        if (fepi) {
            // the residual tile -> the P tiles (every P.V MMA has completed: free), 32-column SW64
            // boxes of 8 KB; O (* 1/l) + residual -> bf16 in place; whole 8-row groups leave by TMA
            // (rows of a neighbouring run are never written), a run's < 8 trailing rows by 16-byte
            // stores
            unsigned char* rt = ptile;
            const uint32_t rts = smem_u32(rt);
            const int nbox = dvs >> 5;
            if (tid == 0) {
                arrive_expect_tx(res_bar, (uint32_t)(nbox * 8192));
                for (int bx = 0; bx < nbox; bx++) tma2d(rts + bx * 8192, &tr, c0 + bx * 32, m0, res_bar);
            }
            mbar_wait(res_bar, 0);
#pragma unroll 1
            for (int cb = 0; cb < dvs; cb += 32) {
                tmem_ld32(tmem + lane_off + O_COL + cb, v);
                unsigned char* bp = rt + (cb >> 5) * 8192 + lr * 64;
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    uint4* pp = (uint4*)(bp + ((j ^ ((lr >> 1) & 3)) << 4));
                    uint4 rr = *pp;
                    uint32_t* h = (uint32_t*)&rr;
#pragma unroll
                    for (int e2 = 0; e2 < 4; e2++) {
                        const float lo = __uint_as_float(h[e2] << 16), hi = __uint_as_float(h[e2] & 0xffff0000u);
                        const __nv_bfloat162 o2 = __floats2bfloat162_rn(__fadd_rn(v[8 * j + 2 * e2] * inv_l, lo),
                                                                        __fadd_rn(v[8 * j + 2 * e2 + 1] * inv_l, hi));
                        h[e2] = *(const uint32_t*)&o2;
                    }
                    *pp = rr;
                }
            }
            fence_async_smem();
            asm volatile("bar.sync 3, 128;" ::: "memory");
            const int rows = min(128, q_end - m0), g8 = rows >> 3;
            if (tid == 0) {
                if (g8 > 0) {
                    for (int bx = 0; bx < nbox; bx++) {
                        if (g8 == 16) {
                            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&to),
                                         "r"(c0 + bx * 32), "r"(m0), "r"(rts + bx * 8192)
                                         : "memory");
                        } else {
                            for (int g = 0; g < g8; g++)
                                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&to8),
                                             "r"(c0 + bx * 32), "r"(m0 + g * 8), "r"(rts + bx * 8192 + g * 512)
                                             : "memory");
                        }
                    }
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
            const int r0 = g8 * 8, upr = dvs >> 3, total = (rows - r0) * upr;
            if (total > 0) {
                __nv_bfloat16* orow = (__nv_bfloat16*)ref_base(a.out, t) + (long long)(m0 + r0) * a.out.ld + c0;
                for (int i = tid; i < total; i += 128) {
                    const int rr_ = i / upr, un = i - rr_ * upr, r = r0 + rr_, j = un & 3;
                    const uint4 val = *(const uint4*)(rt + (un >> 2) * 8192 + r * 64 + ((j ^ ((r >> 1) & 3)) << 4));
                    *(uint4*)(orow + (long long)rr_ * a.out.ld + un * 8) = val;
                }
            }
            if (tid == 0 && g8 > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem read before exit
        } else {
            float* ost = (float*)smem;
#pragma unroll 1
            for (int cb = 0; cb < dvs; cb += 32) {
                tmem_ld32(tmem + lane_off + O_COL + cb, v);
                if (onepass) {
#pragma unroll
                    for (int q = 0; q < 32; q++) v[q] *= inv_l;
                }
#pragma unroll
                for (int q = 0; q < 8; q++)
                    *(float4*)(ost + lr * EPI_LD + cb + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            }
        }
    }
    if (dsp && warp >= 4) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (pmode != P_OUT && !splitkv && !fepi) {
        // all six warps: residual + O -> out, 16-column chunks columns-fastest (coalesced 16-byte runs);
        // each thread first issues the residual loads of EB chunks, then adds and stores them, so the
        // L2 round trips overlap (one per chunk serialised ~0.5 us each: 16 chunks per thread at
        // dvs = 256 made the epilogue ~9 us)
        asm volatile("bar.sync 2, 192;" ::: "memory");
        const float* ost = (const float*)smem;
        char* ob = ref_base(a.out, t);
        char* pbp = a.pre.ptr ? ref_base(a.pre, t) : nullptr;
        const char* rb = a.res.ptr ? ref_base(a.res, t) : nullptr;
        const bool fast = (!rb || (a.res.dtype == FIS_BF16 && (a.res.ld % 8) == 0 && (((uintptr_t)rb) & 15) == 0)) &&
                          a.out.dtype == FIS_BF16 && (a.out.ld % 8) == 0 && (((uintptr_t)ob) & 15) == 0 && !pbp &&
                          (a.dv % 16) == 0;
        const int chunks = dvs / 16;
        const int nrows = min(128, q_end - m0), total = nrows * chunks;
        constexpr int EB = 6;
#pragma unroll 1
        for (int i0 = tid; i0 < total; i0 += THREADS * EB) {
            if (fast) {
                uint4 rr[EB][2];
#pragma unroll
                for (int e = 0; e < EB; e++) {
                    const int item = i0 + e * THREADS;
                    rr[e][0] = rr[e][1] = make_uint4(0u, 0u, 0u, 0u);
                    if (rb && item < total) {
                        const __nv_bfloat16* p = (const __nv_bfloat16*)rb +
                                                 (long long)(m0 + item / chunks) * a.res.ld + c0 + (item % chunks) * 16;
                        rr[e][0] = FIS_LD_U4(p);
                        rr[e][1] = FIS_LD_U4(p + 8);
                    }
                }
#pragma unroll
                for (int e = 0; e < EB; e++) {
                    const int item = i0 + e * THREADS;
                    if (item >= total) break;
                    const int rr_ = item / chunks, cc = (item % chunks) * 16;
                    const float* src = ost + rr_ * EPI_LD + cc;
                    const __nv_bfloat162* hr = (const __nv_bfloat162*)rr[e];
                    uint4 o[2];
                    __nv_bfloat162* ho = (__nv_bfloat162*)o;
#pragma unroll
                    for (int k4 = 0; k4 < 4; k4++) {
                        const float4 f = *(const float4*)(src + 4 * k4);
                        const float2 r0 = __bfloat1622float2(hr[2 * k4]), r1 = __bfloat1622float2(hr[2 * k4 + 1]);
                        ho[2 * k4] = __floats2bfloat162_rn(__fadd_rn(f.x, r0.x), __fadd_rn(f.y, r0.y));
                        ho[2 * k4 + 1] = __floats2bfloat162_rn(__fadd_rn(f.z, r1.x), __fadd_rn(f.w, r1.y));
                    }
                    uint4* dst = (uint4*)((__nv_bfloat16*)ob + (long long)(m0 + rr_) * a.out.ld + c0 + cc);
                    dst[0] = o[0];
                    dst[1] = o[1];
                }
            } else {
                for (int e = 0; e < EB; e++) {
                    const int item = i0 + e * THREADS;
                    if (item >= total) break;
                    const int rr_ = item / chunks, cc = (item % chunks) * 16;
                    const int n = c0 + cc, row = m0 + rr_;
                    const int nvalid = min(16, a.dv - n);
                    if (nvalid <= 0) continue;
                    float w[16];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const float4 f = *(const float4*)(ost + rr_ * EPI_LD + cc + 4 * q);
                        w[4 * q] = f.x; w[4 * q + 1] = f.y; w[4 * q + 2] = f.z; w[4 * q + 3] = f.w;
                    }
                    if (pbp) store_row16(pbp, a.pre.dtype, (long long)row * a.pre.ld + n, nvalid, w);
                    if (rb) {
                        float q[16];
                        load_row16(rb, a.res.dtype, (long long)row * a.res.ld + n, nvalid, q);
#pragma unroll
                        for (int e2 = 0; e2 < 16; e2++) w[e2] = __fadd_rn(w[e2], q[e2]);
                    }
                    store_row16(ob, a.out.dtype, (long long)row * a.out.ld + n, nvalid, w);
                }
            }
        }
    }
    goto done;
ks_softmax : {
        // key split (P_OUT_KS): statistics of this CTA's key block, exchange with the peer block's
        // through DSMEM, then P of this block from the same (resident) S
        const int lr = tid, r = m0 + lr;
        const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
        const float sl = a.scale * 1.4426950408889634f;
        float mrow = -INFINITY, lrow = 0.f;
        float v[32];
        if (!idle) {
            mbar_wait(s_ready, 0);
            tc_fence_after();
#pragma unroll 1
            for (int cb = 0; cb < 128; cb += 32) {
                tmem_ld32(trow + cb, v);
                const int lim = n_keys - cb;
                float cm = -INFINITY;
#pragma unroll
                for (int q = 0; q < 32; q++)
                    if (q < lim) cm = fmaxf(cm, v[q]);
                const float mn = fmaxf(mrow, cm * sl);
                float add = 0.f;
#pragma unroll
                for (int q = 0; q < 32; q++)
                    if (q < lim) add += ex2(fmaf(v[q], sl, -mn));
                lrow = (mrow == -INFINITY ? 0.f : lrow * ex2(mrow - mn)) + add;
                mrow = mn;
            }
        }
        xst[lr] = make_float2(mrow, lrow);
        cluster_sync_all();  // phase 1: both blocks' statistics written
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(xst + lr)), "r"((int)blockIdx.x ^ 1));
        float pm, pl;
        asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(pm), "=f"(pl) : "r"(ra) : "memory");
        const float M = fmaxf(mrow, pm);
        const float Ls = (mrow == -INFINITY ? 0.f : lrow * ex2(mrow - M)) + (pm == -INFINITY ? 0.f : pl * ex2(pm - M));
        if (!idle) {
            const float off = M + __log2f(Ls);
            __nv_bfloat16* prow = (__nv_bfloat16*)a.ws + (long long)r * pw + kb_off;
#pragma unroll 1
            for (int cb = 0; cb < 128; cb += 32) {
                tmem_ld32(trow + cb, v);
                const int lim = n_keys - cb;
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    uint4 pk;
                    __nv_bfloat162* h = (__nv_bfloat162*)&pk;
#pragma unroll
                    for (int e2 = 0; e2 < 4; e2++) {
                        const int q0 = 8 * u + 2 * e2;
                        const float p0 = q0 < lim ? ex2(fmaf(v[q0], sl, -off)) : 0.f;
                        const float p1 = q0 + 1 < lim ? ex2(fmaf(v[q0 + 1], sl, -off)) : 0.f;
                        h[e2] = __floats2bfloat162_rn(p0, p1);
                    }
                    if (r < q_end) *(uint4*)(prow + cb + 8 * u) = pk;
                }
            }
        }
        cluster_sync_all();  // phase 2: the peer has read our statistics
        goto teardown;
    }
done:
    if (ks) {  // producer / MMA warps (and an idle CTA's) take part in both cluster phases
        cluster_sync_all();
        cluster_sync_all();
    }
teardown:
    tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    ltr(ls, 7);
}

}  // namespace attn
}  // namespace fis

FIS_LTR_SETTER(fis_ltr_set_attn)

// value-slice width: largest multiple of 32 dividing dv with <= 256 columns
static int attn_slice(int dv) {
    for (int w = 256; w >= 32; w -= 32)
        if (dv % w == 0) return w;
    return 0;
}

// P sharing (P_OUT + P_IN launches) for this call? Long key runs trade one extra serial launch for
// 1/slices of the S work, which pays only when the grid has CTAs to spare (stacked requests).
static bool attn_share(const fis_attn_args* a, int dvs) {
    static int share_off = getenv("FIS_ATTN_SHARE") && getenv("FIS_ATTN_SHARE")[0] == '0';
    const long long pw = ((long long)a->max_seg_k + 127) / 128 * 128;
    const long long ctas = (long long)(a->dv / dvs) * (((a->nseg > 0 ? a->max_seg_q : a->m) + 127) / 128) *
                           (a->nseg > 0 ? a->nseg : 1);
    const int slices = a->dv / dvs;
    if (share_off || a->max_seg_k <= 0 || a->max_seg_k > 4096 || slices < 2 || !a->ws ||
        a->ws_bytes < (long long)a->m * pw * 2)
        return false;
    // batch 1 (a grid smaller than the GPU): the slices' redundant S work runs in parallel anyway,
    // a second (serial) launch only adds latency (r01 C2 step: 1.358 ms unshared vs 1.390 shared)
    // (r02: forcing it for the d = 1280 levels measured 27.6 vs 29.1 us for L2 self attention,
    // but more for cross attention; a wash at the step level)
    if (ctas < 148) return false;
    // runs of >= 3 key blocks over <= 2 value slices: the one-pass kernel (no statistics pass)
    // recomputes S once per slice, cheaper than P_OUT's two S passes + the P_IN launch (r02, R = 64:
    // L0 self attention 131 -> 113 us; at 5 slices sharing still wins)
    if (slices <= 2 && a->max_seg_k > 256) return false;
    // one key block: recomputing S per slice is cheap unless the head dim is large (r01: L0 cross
    // attention 23 + 48 us shared vs one launch unshared)
    if (a->max_seg_k <= 128) return (long long)a->d * (slices - 1) >= 1280;
    return a->max_seg_k <= 256 || ctas >= 2 * 148;
}

// d-split (P_DSPLIT) for this call? Batch-1 runs of <= 128 keys whose grid leaves the GPU mostly
// idle: the cs = dv / dvs value-slice CTAs of a query tile share the S reduction (<= 4 d chunks
// each) instead of each computing all of it.
static bool attn_dsplit(const fis_attn_args* a, int dvs) {
    static int off = getenv("FIS_ATTN_DSPLIT") && getenv("FIS_ATTN_DSPLIT")[0] == '0';
    const int cs = a->dv / dvs, dch = a->d / 64;
    // (d >= 1024: at d = 320 / 640 the exchange costs what the split saves, r02 step tables)
    if (off || a->nseg > 0 || a->n_keys > 256 || cs < 2 || cs > 8 || dch < 16 || (dch + cs - 1) / cs > 4) return false;
    const int rp = (128 + cs - 1) / cs;
    if (a->n_keys > 128 && rp > 32) return false;  // two key blocks: one owned-row iteration
    if ((cs - 1) * rp * 512 > fis::attn::P_BYTES + fis::attn::RX_EXTRA) return false;
    return (long long)cs * ((a->m + 127) / 128) < 148;
}

// Split-KV factor for batch-1 runs of >= 8 key blocks whose grid leaves most SMs idle: the
// largest split with >= 2 key blocks per CTA that keeps the grid within one wave (<= 8), if the
// workspace holds the partials (the caller sizes it: fis_attn_ws_bytes).
static int attn_kv_splits(const fis_attn_args* a, int dvs) {
    static int off = getenv("FIS_ATTN_SPLITKV") && getenv("FIS_ATTN_SPLITKV")[0] == '0';
    const int nkb = (a->n_keys + 127) / 128;
    // runs of >= 8 key blocks: the split CTAs merge their own rows after a group barrier; on
    // shorter runs the partial round trip costs more than the split saves (r02, C2 batch 1 / dense
    // step: 400 keys 18 -> 23.5 us, 1024 keys 40 -> 26-32 us, 4096 keys 88 -> 60 us)
    if (off || a->nseg > 0 || nkb < 8 || !a->ws) return 1;
    const int slices = a->dv / dvs, tiles = (a->m + 127) / 128;
    const long long ctas = (long long)slices * tiles;
    if (ctas > 512) return 1;  // counter slots (2 per group)
    int kvs = (int)(148 / ctas);
    if (kvs > nkb / 2) kvs = nkb / 2;
    if (kvs > 8) kvs = 8;
    if (kvs < 2) return 1;
    const int kvper = (nkb + kvs - 1) / kvs;
    kvs = (nkb + kvper - 1) / kvper;  // every split owns >= 1 block
    const long long need = ctas * kvs * 128 * (dvs + 4) * 4 + 4096;
    return need <= a->ws_bytes ? kvs : 1;
}

// Workspace bytes a fis_attn call can use (P sharing scratch or split-KV partials + counters).
// Split-KV grids stay within one wave (<= 148 CTAs of 128 rows x <= 256 + 4 floats).
extern "C" long long fis_attn_ws_bytes(int m, int max_keys, int dv) {
    const long long mp = (m + 127) / 128 * 128, pw = (max_keys + 127) / 128 * 128;
    const long long p = mp * pw * 2, kv = 148ll * 128 * ((dv < 256 ? dv : 256) + 4) * 4;
    return (p > kv ? p : kv) + 4096;
}

int fis_attn_short_ok(const fis_attn_args* a);                      // fis_attn_short.cu
int fis_attn_short_launch(const fis_attn_args* a, cudaStream_t stream);

// Kernel launches one fis_attn call makes (1, or 2 when the value slices share P); 0 = unsupported.
extern "C" int fis_attn_launches(const fis_attn_args* a) {
    const int dvs = attn_slice(a->dv);
    if (!dvs) return 0;
    if (fis_attn_short_ok(a)) return 1;
    return attn_share(a, dvs) ? 2 : 1;
}

// Q [m][d], K [n_keys][d] (with segments: n_keys = rows of K), V^T [dv][>= n_keys]; bf16, rows
// 16-byte aligned, no per-step stride (scratch activations / per-edit text K/V).
extern "C" int fis_attn(const fis_attn_args* a, void* stream) {
    if (a->m == 0) return FIS_OK;
    if (a->d % 64 || a->n_keys < 1 || a->q.dtype != FIS_BF16 || a->k.dtype != FIS_BF16 || a->vt.dtype != FIS_BF16 ||
        (a->q.ld % 8) || (a->k.ld % 8) || (a->vt.ld % 8) || a->q.step_stride || a->k.step_stride ||
        a->vt.step_stride)
        return FIS_ERR_UNSUPPORTED;
    const int dvs = attn_slice(a->dv);
    if (!dvs) return FIS_ERR_UNSUPPORTED;
    {  // every key run <= 256 keys on a large grid: the persistent short-run kernel
        const int r = fis_attn_short_launch(a, (cudaStream_t)stream);
        if (r >= 0) return r;
    }
    CUtensorMap tq, tk, tv, tp;
    if (!encode_2d(&tq, a->q.ptr, a->m, a->d, a->q.ld, 128) ||
        !encode_2d(&tk, a->k.ptr, a->n_keys, a->d, a->k.ld, 128) ||
        !encode_2d(&tv, a->vt.ptr, a->dv, a->n_keys, a->vt.ld, dvs))
        return FIS_ERR_UNSUPPORTED;
    const long long pw = ((long long)a->max_seg_k + 127) / 128 * 128;
    const bool share = attn_share(a, dvs) && encode_2d(&tp, a->ws, a->m, pw, pw, 128);
    if (!share) std::memset(&tp, 0, sizeof(tp));
    // TMA residual / output epilogue (P_FEPI) when both are step-invariant bf16 matrices
    CUtensorMap tr, to, to8;
    static int fepi_off = getenv("FIS_ATTN_FEPI") && getenv("FIS_ATTN_FEPI")[0] == '0';
    int fepi = 0;
    if (!fepi_off && !a->pre.ptr && a->res.ptr && a->res.dtype == FIS_BF16 && !a->res.step_stride &&
        a->out.dtype == FIS_BF16 && !a->out.step_stride && (a->dv % 32) == 0 &&
        encode_2d_sw64(&tr, a->res.ptr, a->m, a->dv, a->res.ld, 128) &&
        encode_2d_sw64(&to, a->out.ptr, a->m, a->dv, a->out.ld, 128) &&
        encode_2d_sw64(&to8, a->out.ptr, a->m, a->dv, a->out.ld, 8))
        fepi = fis::attn::P_FEPI;
    if (!fepi) {
        std::memset(&tr, 0, sizeof(tr));
        std::memset(&to, 0, sizeof(to));
        std::memset(&to8, 0, sizeof(to8));
    }
    static bool configured = false;
    if (!configured) {
        if (cudaFuncSetAttribute(fis::attn::attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 fis::attn::SMEM) != cudaSuccess)
            return FIS_ERR_UNSUPPORTED;
        configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    const dim3 grid = a->nseg > 0 ? dim3(a->dv / dvs, (a->max_seg_q + 127) / 128, a->nseg)
                                  : dim3(a->dv / dvs, (a->m + 127) / 128, 1);
    cfg.blockDim = dim3(fis::attn::THREADS);
    cfg.dynamicSmemBytes = fis::attn::SMEM;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = fis_pdl_enabled() ? 1 : 0;
    if (share) {  // P once per query tile (slice 0), then every slice's P.V from the scratch
        static int ks_off = getenv("FIS_ATTN_KSPLIT") && getenv("FIS_ATTN_KSPLIT")[0] == '0';
        const bool ksplit = !ks_off && a->max_seg_k > 128 && a->max_seg_k <= 256;
        cudaLaunchAttribute at2[2];
        at2[0] = attr[0];
        at2[1].id = cudaLaunchAttributeClusterDimension;
        at2[1].val.clusterDim.x = 2;
        at2[1].val.clusterDim.y = 1;
        at2[1].val.clusterDim.z = 1;
        cfg.gridDim = dim3(ksplit ? 2 : 1, grid.y, grid.z);
        if (ksplit) {  // two key blocks over a 2-CTA cluster
            cfg.attrs = at2;
            cfg.numAttrs = 2;
            if (!fis_pdl_enabled()) {
                cfg.attrs = at2 + 1;
                cfg.numAttrs = 1;
            }
        }
        if (cudaLaunchKernelEx(&cfg, fis::attn::attn_kernel, *a, tq, tk, tv, tp, tr, to, to8, dvs,
                               (int)(ksplit ? fis::attn::P_OUT_KS : fis::attn::P_OUT)) != cudaSuccess)
            return FIS_ERR_LAUNCH;
        cfg.attrs = attr;
        cfg.numAttrs = fis_pdl_enabled() ? 1 : 0;
    }
    cfg.gridDim = grid;
    if (!share && attn_dsplit(a, dvs)) {  // the value slices of a query tile = one cluster
        cudaLaunchAttribute at2[2];
        at2[0] = attr[0];
        at2[1].id = cudaLaunchAttributeClusterDimension;
        at2[1].val.clusterDim.x = grid.x;
        at2[1].val.clusterDim.y = 1;
        at2[1].val.clusterDim.z = 1;
        cfg.attrs = fis_pdl_enabled() ? at2 : at2 + 1;
        cfg.numAttrs = fis_pdl_enabled() ? 2 : 1;
        return cudaLaunchKernelEx(&cfg, fis::attn::attn_kernel, *a, tq, tk, tv, tp, tr, to, to8, dvs, (int)fis::attn::P_DSPLIT | fepi) ==
                       cudaSuccess
                   ? FIS_OK : FIS_ERR_LAUNCH;
    }
    static int onepass_off = getenv("FIS_ATTN_ONEPASS") && getenv("FIS_ATTN_ONEPASS")[0] == '0';
    if (!share && !onepass_off) {
        const int kvs = attn_kv_splits(a, dvs);
        if (kvs > 1) {
            // the split CTAs of a group meet at a barrier before merging: a cooperative launch makes
            // the whole grid co-resident (a spinning grid could otherwise hold SMs that the rest of
            // its CTAs -- or another spinning grid on a concurrent stream -- wait for)
            cudaLaunchConfig_t c2 = cfg;
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = 1;
            at[1] = attr[0];
            c2.attrs = at;
            c2.numAttrs = fis_pdl_enabled() ? 2 : 1;
            c2.gridDim = dim3(grid.x, grid.y, kvs);
            if (cudaLaunchKernelEx(&c2, fis::attn::attn_kernel, *a, tq, tk, tv, tp, tr, to, to8, dvs,
                                   (int)fis::attn::P_NONE | fis::attn::P_ONEPASS_OK | fis::attn::P_SPLITKV) ==
                cudaSuccess)
                return FIS_OK;
            cudaGetLastError();  // not co-schedulable here: the unsplit kernel below
        }
    }
    return cudaLaunchKernelEx(&cfg, fis::attn::attn_kernel, *a, tq, tk, tv, tp, tr, to, to8, dvs,
                              (share ? (int)fis::attn::P_IN
                                     : (int)fis::attn::P_NONE | (onepass_off ? 0 : fis::attn::P_ONEPASS_OK)) | fepi) ==
                   cudaSuccess
               ? FIS_OK : FIS_ERR_LAUNCH;
}
