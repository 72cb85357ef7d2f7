// SPDX-License-Identifier: Apache-2.0
//
// Component-level kernels behind the reference's free-standing API
// (/root/reference/proj/include/pikv): KVStore::insert / retrieve / erase
// (kvstore.cpp:107-185), the scheduler's score_entry / observe_hits /
// adakv_update (scheduler.cpp:181-229, 332-342), the router's record_miss /
// adapt (router.cpp:236-255), attention over stored entries
// (pipeline.cpp:59-85) and the codec's encode_vector / decode_vector
// (compressor.cpp:364-474).  They act on one stream of an engine -- the same
// HBM store, router and scheduler state Engine::step uses -- so a caller of
// the component API and of the decode step see one consistent state.
//
// These are the reference's one-entry / one-call granularity: single-CTA
// kernels for the sequential mutations (the reference's order is the
// contract), grid-wide kernels and a device radix sort where the work is a
// scan (retrieve).  The decode hot path does not use them.
#include <cub/cub.cuh>

#include "pikv_dev.cuh"

namespace pikv_dev {

// Page-record append for an entry with arbitrary metadata (rec_append with
// the entry's own last_access / freq).
__device__ __forceinline__ void rec_add(const Dims& D, const State& S, int64_t ring, uint64_t sq, uint64_t la,
                                        uint64_t fr) {
    const int64_t r = page_rec(D, ring, sq);
    if (S.pr_cnt[r] == 0) {
        atomicAdd(&S.pages_live[ring / D.SPD], 1);
        S.pr_cnt[r] = 1;
        S.pr_first[r] = (int)(sq % (uint64_t)D.page_size);
        S.pr_sla[r] = la;
        S.pr_sf[r] = fr;
    } else {
        S.pr_cnt[r] += 1;
        S.pr_sla[r] += la;
        S.pr_sf[r] += fr;
    }
}

// Stored value of element c of a pool entry half (row 0 = K, 1 = V) as fp32.
__device__ __forceinline__ float entry_value(const Dims& D, const uint8_t* ent, int row, int c) {
    const uint8_t* p = ent + (int64_t)row * D.payload_bytes;
    if (D.codec == PIKV_CODEC_INT8 || D.codec == PIKV_CODEC_INT4) {
        const float sc = ((const float*)(ent + 2 * D.payload_bytes))[row * D.H + c / D.dph];
        int code;
        if (D.codec == PIKV_CODEC_INT8) {
            code = (int)((const int8_t*)p)[c];
        } else {
            const int nib = (p[c >> 1] >> ((c & 1) * 4)) & 0xF;
            code = nib >= 8 ? nib - 16 : nib;
        }
        return __fmul_rn((float)code, sc);
    }
    if (D.kv_dtype == PIKV_DTYPE_BF16) return __uint_as_float(((uint32_t)((const uint16_t*)p)[c]) << 16);
    return ((const float*)p)[c];
}

// Store one d'-wide row (fp32, already in the stored space) into a pool entry
// half: kv_dtype values, or per-head symmetric absmax codes (the engine's
// quantizer, encode_row / oracle po_quantize_row).
__device__ void store_row(const Dims& D, const float* __restrict__ x, uint8_t* ent, int row) {
    const int tid = threadIdx.x, nt = blockDim.x;
    uint8_t* dst = ent + (int64_t)row * D.payload_bytes;
    if (D.codec != PIKV_CODEC_INT8 && D.codec != PIKV_CODEC_INT4) {
        for (int c = tid; c < D.dp; c += nt) {
            if (D.kv_dtype == PIKV_DTYPE_BF16) ((uint16_t*)dst)[c] = f32_to_bf16_rne(x[c]);
            else ((float*)dst)[c] = x[c];
        }
        return;
    }
    const int bits = D.codec == PIKV_CODEC_INT8 ? 8 : 4, hw = D.dph;
    const float qmax = bits == 8 ? 127.0f : 7.0f;
    float* scales = (float*)(ent + 2 * D.payload_bytes) + row * D.H;
    const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
    for (int h = warp; h < D.H; h += nw) {
        float amax = 0.f;
        for (int i = lane; i < hw; i += 32) amax = fmaxf(amax, fabsf(x[h * hw + i]));
        for (int off = 16; off; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
        float inv = 0.f, scale = 0.f;
        if (amax > 0.f) scale = __fdiv_rn(amax, qmax), inv = __fdiv_rn(qmax, amax);
        if (lane == 0) scales[h] = scale;
        if (bits == 8) {
            for (int i = lane; i < hw; i += 32) {
                const float c = fminf(fmaxf(rintf(__fmul_rn(x[h * hw + i], inv)), -qmax), qmax);
                ((int8_t*)dst)[h * hw + i] = (int8_t)(int)c;
            }
        } else {
            for (int i2 = lane; i2 < hw / 2; i2 += 32) {
                const float c0 = fminf(fmaxf(rintf(__fmul_rn(x[h * hw + 2 * i2], inv)), -qmax), qmax);
                const float c1 = fminf(fmaxf(rintf(__fmul_rn(x[h * hw + 2 * i2 + 1], inv)), -qmax), qmax);
                dst[(h * hw) / 2 + i2] = (uint8_t)(((int)c0 & 0xF) | (((int)c1 & 0xF) << 4));
            }
        }
    }
}

// ---------------------------------------------------------------------------
// KVStore::insert (kvstore.cpp:107-120) + ShardBuffer::insert (36-53) of n
// entries, in order, into stream s.  One CTA; thread 0 does the bookkeeping,
// all threads move payloads.  A displaced entry (ring full) comes back with
// its metadata and decoded K/V.  status: 0 ok, else the PIKV_ERR_* of the
// first failing entry (pool exhausted: the entries before it stay inserted,
// as n separate insert calls would).
__global__ void k_store_insert(Dims D, State S, int s, int n, const pikv_entry* __restrict__ in,
                               const float* __restrict__ kv, const double* __restrict__ layers,
                               pikv_entry* __restrict__ disp, float* __restrict__ disp_kv,
                               double* __restrict__ disp_layers, int32_t* __restrict__ disp_flag,
                               int32_t* __restrict__ status) {
    __shared__ int64_t sm_ring, sm_gi, sm_dst;
    __shared__ int sm_ok, sm_disp, sm_slot;
    const int tid = threadIdx.x;
    if (tid == 0) *status = 0;
    for (int j = 0; j < n; ++j) {
        if (tid == 0) {
            const pikv_entry e = in[j];
            const int raw = shard_raw(e.token_id, e.expert_id, D.n_tok, D.n_exp, D.additive);
            const int dev = raw % D.G, sh = raw / D.G;
            const int64_t ring = (int64_t)s * D.R + (int64_t)dev * D.SPD + sh;  // world 1 (host-checked)
            const int slot = S.head[ring];
            const int64_t gi = ring * D.S + slot;
            const int64_t pidx = ring * D.ppr + slot / D.spg;
            int32_t page = S.page_table[pidx];
            const bool dsp = S.id[gi] != 0;
            sm_ok = 1;
            if (!dsp && page < 0) {  // a fresh storage page from the pool
                const int top = *S.free_top - 1;
                if (top < 0) {
                    sm_ok = 0;
                    *status = PIKV_ERR_OUT_OF_MEMORY;
                } else {
                    *S.free_top = top;
                    page = S.free_stack[top];
                    S.page_table[pidx] = page;
                    S.page_live[page] = 0;
                }
            }
            sm_ring = ring, sm_gi = gi, sm_slot = slot, sm_disp = dsp;
            sm_dst = (int64_t)page * D.spg + slot % D.spg;
        }
        __syncthreads();
        if (!sm_ok) return;
        const int64_t ring = sm_ring, gi = sm_gi;
        uint8_t* ent = S.pool + sm_dst * (int64_t)D.entry_bytes;
        if (sm_disp) {  // the displaced entry leaves with its payload (kvstore.hpp:106-108)
            for (int o = tid; o < 2 * D.dp; o += blockDim.x)
                disp_kv[((int64_t)j * 2 + o / D.dp) * D.dp + o % D.dp] = entry_value(D, ent, o / D.dp, o % D.dp);
            for (int l = tid; l < D.n_layers; l += blockDim.x)
                if (disp_layers) disp_layers[(int64_t)j * D.n_layers + l] = S.per_layer[gi * D.n_layers + l];
        }
        __syncthreads();
        if (tid == 0) {
            disp_flag[j] = sm_disp;
            if (sm_disp) {
                pikv_entry o;
                o.id = S.id[gi];
                o.shard_seq = S.shard_seq[gi];
                o.token_id = S.token[gi];
                o.expert_id = S.expert[gi];
                o.has_layers = S.has_pl[gi];
                o.insert_step = S.insert_step[gi];
                o.last_access_step = S.last_access[gi];
                o.freq = S.freq[gi];
                o.attn_mass = S.attn_mass[gi];
                disp[j] = o;
                rec_drop_front(D, S, ring, o.shard_seq, o.last_access_step, o.freq);
                S.st_overwrites[s] += 1;
            } else {
                S.live[ring] += 1;
                S.page_live[S.page_table[ring * D.ppr + sm_slot / D.spg]] += 1;
            }
            const pikv_entry e = in[j];
            const uint64_t sq = S.seq[ring]++;
            S.id[gi] = S.next_id[s]++;
            S.shard_seq[gi] = sq;
            S.token[gi] = e.token_id;
            S.expert[gi] = e.expert_id;
            S.insert_step[gi] = e.insert_step;
            S.last_access[gi] = e.last_access_step;
            S.freq[gi] = e.freq;
            S.attn_mass[gi] = e.attn_mass;
            S.has_pl[gi] = layers != nullptr && e.has_layers && D.n_layers > 0;
            for (int l = 0; l < D.n_layers; ++l)
                S.per_layer[gi * D.n_layers + l] = S.has_pl[gi] ? layers[(int64_t)j * D.n_layers + l] : 0.0;
            rec_add(D, S, ring, sq, e.last_access_step, e.freq);
            S.head[ring] = (sm_slot + 1) % D.S;
            S.st_inserts[s] += 1;
        }
        store_row(D, kv + (int64_t)j * 2 * D.dp, ent, 0);
        store_row(D, kv + ((int64_t)j * 2 + 1) * D.dp, ent, 1);
        __syncthreads();
    }
}

// KVStore::erase (kvstore.cpp:180-185): the live entry with this id, if any.
// The page record keeps count / sums; its first member advances past holes
// (D.holes is set by the caller).  *status = 1 when erased.
__global__ void k_store_erase(Dims D, State S, int s, uint64_t id, int32_t* __restrict__ status) {
    __shared__ long long sm_gi;
    if (threadIdx.x == 0) sm_gi = -1;
    __syncthreads();
    const int64_t n = (int64_t)D.R * D.S, base = (int64_t)s * n;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        if (S.id[base + i] == id) sm_gi = base + i;  // ids are unique
    __syncthreads();
    if (threadIdx.x != 0) return;
    const int64_t gi = sm_gi;
    *status = gi >= 0;
    if (gi < 0) return;
    const int64_t ring = gi / D.S;
    const int slot = (int)(gi % D.S);
    const uint64_t sq = S.shard_seq[gi];
    S.id[gi] = 0;
    S.live[ring] -= 1;
    const int64_t pt_i = ring * D.ppr + slot / D.spg;
    const int32_t page = S.page_table[pt_i];
    if (--S.page_live[page] == 0) {  // storage page empty: back to the pool
        S.page_table[pt_i] = -1;
        S.free_stack[(*S.free_top)++] = page;
    }
    const int64_t r = page_rec(D, ring, sq);
    const int off = (int)(sq % (uint64_t)D.page_size);
    S.pr_sla[r] -= S.last_access[gi];
    S.pr_sf[r] -= S.freq[gi];
    if (--S.pr_cnt[r] == 0) {
        atomicSub(&S.pages_live[ring / D.SPD], 1);
        S.pr_first[r] = 0, S.pr_sla[r] = 0, S.pr_sf[r] = 0;
    } else if (off == S.pr_first[r]) {
        S.pr_first[r] = next_member(D, S, ring, sq / (uint64_t)D.page_size, off + 1);
    }
}

// KVStore::retrieve (kvstore.cpp:122-178), pass 1: the stream's live entries
// with expert in the set and token < since get the key token << 8 | expert
// (E <= 256), all others the max key; vals = stream-local slot index.
__global__ void k_cretr_keys(Dims D, State S, int s, int64_t since, const uint32_t* __restrict__ want,
                             uint64_t* __restrict__ keys, int32_t* __restrict__ vals, int32_t* __restrict__ cnt) {
    const int64_t n = (int64_t)D.R * D.S, base = (int64_t)s * n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t gi = base + i;
        bool hit = false;
        if (S.id[gi] != 0) {
            const int e = S.expert[gi];
            hit = S.token[gi] < since && e >= 0 && e < 256 && ((want[e >> 5] >> (e & 31)) & 1u);
        }
        keys[i] = hit ? ((uint64_t)S.token[gi] << 8) | (uint64_t)S.expert[gi] : ~0ull;
        vals[i] = (int32_t)i;
        if (hit) atomicAdd(cnt, 1);
    }
}

// pass 3 (after the sort): the meta bump of every hit (freq += 1,
// last_access = now; kvstore.cpp:164-168) with its page record, and the hit
// count per expert (misses).
__global__ void k_cretr_bump(Dims D, State S, int s, uint64_t now, const int32_t* __restrict__ sorted,
                             const int32_t* __restrict__ cnt, uint32_t* __restrict__ found) {
    const int n = *cnt;
    const int64_t base = (int64_t)s * D.R * D.S;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int64_t gi = base + sorted[i];
        const int64_t ring = gi / D.S;
        const uint64_t la = S.last_access[gi];
        S.last_access[gi] = now;
        S.freq[gi] += 1;
        const int64_t r = page_rec(D, ring, S.shard_seq[gi]);
        atomicAdd((unsigned long long*)&S.pr_sla[r], (unsigned long long)(now - la));
        atomicAdd((unsigned long long*)&S.pr_sf[r], 1ull);
        atomicAdd(&found[S.expert[gi]], 1u);
    }
}

// score_entry (scheduler.cpp:181-229) on caller-given entry metadata.
__global__ void k_score_meta(Cfg C, const pikv_entry* __restrict__ m, const double* __restrict__ layers,
                             int n_layers, int n, uint64_t now, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    struct Given {
        pikv_entry e;
        const double* p;
        __device__ uint64_t ins() const { return e.insert_step; }
        __device__ uint64_t la() const { return e.last_access_step; }
        __device__ uint64_t freq() const { return e.freq; }
        __device__ double mass() const { return e.attn_mass; }
        __device__ int64_t token() const { return e.token_id; }
        __device__ bool has_pl() const { return e.has_layers && p; }
        __device__ const double* pl() const { return p; }
    } g{m[i], layers ? layers + (int64_t)i * n_layers : nullptr};
    out[i] = score_impl(C, g, n_layers, now);
}

// Scheduler / router state updates of one stream (one thread):
//   op 0 observe_hits (scheduler.cpp:332-338), 1 adakv_update (340-342),
//   2 state.step++ (scheduler.cpp:328), 3 record_miss (router.cpp:236-241),
//   4 adapt (router.cpp:243-255) over experts[0..n).
__global__ void k_state_op(Dims D, Cfg C, State S, int s, int op, uint64_t a, uint64_t b,
                           const int32_t* __restrict__ experts, int n, double reward) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    switch (op) {
        case 0:
            if (b == 0) return;
            S.running_hit[s] = __dadd_rn(__dmul_rn(C.hit_decay, S.running_hit[s]),
                                         __dmul_rn(__dsub_rn(1.0, C.hit_decay), __ddiv_rn((double)a, (double)b)));
            return;
        case 1:
            S.theta[s] = __dadd_rn(S.theta[s], __dmul_rn(C.adakv_step, __dsub_rn(C.target_hit, S.running_hit[s])));
            return;
        case 2:
            S.sstep[s] += 1;
            return;
        case 3:
            S.miss[(int64_t)s * D.E + (int64_t)a] += 1;
            return;
        case 4: {
            double* bias = S.bias + (int64_t)s * D.E;
            double acc = 0.0;
            for (int e = 0; e < D.E; ++e) acc = __dadd_rn(acc, bias[e]);
            const double mean = __ddiv_rn(acc, (double)D.E);
            for (int j = 0; j < n; ++j) {
                const int e = experts[j];
                const double v = __dadd_rn(bias[e], __dmul_rn(C.bandit_step, __dsub_rn(reward, mean)));
                bias[e] = v < -C.bias_cap ? -C.bias_cap : (C.bias_cap < v ? C.bias_cap : v);
            }
            return;
        }
    }
}

// Stored K/V of n slots of stream s as per-head problems: kh/vh [H][n][dph]
// (the layout k_attention takes: head h = query h), fp32.
__global__ void k_read_heads(Dims D, State S, int s, const int64_t* __restrict__ slots, int n,
                             float* __restrict__ kh, float* __restrict__ vh) {
    const int i = blockIdx.x;
    const int64_t ls = slots[i];
    const int64_t ring = (int64_t)s * D.R + ls / D.S;
    const int slot = (int)(ls % D.S);
    const int32_t page = S.page_table[ring * D.ppr + slot / D.spg];
    const bool live = S.id[ring * D.S + slot] != 0 && page >= 0;
    const uint8_t* ent = live ? S.pool + ((int64_t)page * D.spg + slot % D.spg) * D.entry_bytes : nullptr;
    for (int o = threadIdx.x; o < 2 * D.dp; o += blockDim.x) {
        const int row = o / D.dp, c = o % D.dp, h = c / D.dph, j = c % D.dph;
        const float x = live ? entry_value(D, ent, row, c) : 0.f;
        (row ? vh : kh)[((int64_t)h * n + i) * D.dph + j] = x;
    }
}

// alpha_i = mean over heads of the per-head weights.
__global__ void k_head_mean(const float* __restrict__ w, int H, int n, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double a = 0.0;
    for (int h = 0; h < H; ++h) a += (double)w[(int64_t)h * n + i];
    out[i] = (float)(a / H);
}

// Codec::encode_vector / decode_vector for FastV (crop / zero-fill,
// compressor.cpp:396, 449-453) and Prune (gather / scatter of the sorted kept
// coordinates, 398-402, 454-460), per head of width hd -> r.
__global__ void k_codec_select(int decode, int codec, int64_t rows, int heads, int hd, int r,
                               const int32_t* __restrict__ kept, const float* __restrict__ x, float* __restrict__ y) {
    const int64_t n = rows * heads * (decode ? hd : r);
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
        if (!decode) {
            const int64_t row = o / ((int64_t)heads * r);
            const int h = (int)(o / r % heads), j = (int)(o % r);
            const int i = codec == PIKV_CODEC_FASTV ? j : kept[h * r + j];
            y[o] = x[(row * heads + h) * hd + i];
        } else {
            const int64_t row = o / ((int64_t)heads * hd);
            const int h = (int)(o / hd % heads), i = (int)(o % hd);
            float v = 0.f;
            if (codec == PIKV_CODEC_FASTV) {
                if (i < r) v = x[(row * heads + h) * r + i];
            } else {
                for (int j = 0; j < r; ++j)
                    if (kept[h * r + j] == i) v = x[(row * heads + h) * r + j];
            }
            y[o] = v;
        }
    }
}

// Column variance of n calibration rows (Prune's fit statistic,
// compressor.cpp:250-255): mean then mean squared deviation, fp64.
__global__ void k_col_var(const double* __restrict__ x, int n, int d, double* __restrict__ var) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= d) return;
    double m = 0.0;
    for (int i = 0; i < n; ++i) m += x[(int64_t)i * d + c];
    m /= (double)n;
    double v = 0.0;
    for (int i = 0; i < n; ++i) {
        const double t = x[(int64_t)i * d + c] - m;
        v += t * t;
    }
    var[c] = v / (double)(n > 1 ? n : 1);
}

// ---- launchers -------------------------------------------------------------
void launch_store_insert(const Dims& D, const State& S, int s, int n, const pikv_entry* in, const float* kv,
                         const double* layers, pikv_entry* disp, float* disp_kv, double* disp_layers,
                         int32_t* disp_flag, int32_t* status, cudaStream_t st) {
    k_store_insert<<<1, 256, 0, st>>>(D, S, s, n, in, kv, layers, disp, disp_kv, disp_layers, disp_flag, status);
}
void launch_store_erase(const Dims& D, const State& S, int s, uint64_t id, int32_t* status, cudaStream_t st) {
    k_store_erase<<<1, 1024, 0, st>>>(D, S, s, id, status);
}
// retrieve: keys -> device radix sort (cub) -> bump.  scratch: see
// retrieve_scratch_bytes.  sorted_vals gets the hits first, in key order.
size_t retrieve_scratch_bytes(const Dims& D) {
    const int64_t n = (int64_t)D.R * D.S;
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
    return ((tmp + 255) & ~(size_t)255) + 2 * (size_t)n * 8 + 2 * (size_t)n * 4 + 1024 + 256 * 4 + 64;
}
int launch_retrieve(const Dims& D, const State& S, int s, int64_t since, uint64_t now, const uint32_t* want,
                    void* scratch, int32_t** sorted_out, int32_t** cnt_out, uint32_t** found_out, cudaStream_t st) {
    const int64_t n = (int64_t)D.R * D.S;
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
    uint8_t* p = (uint8_t*)scratch;
    void* cub_tmp = p;
    p += (tmp + 255) & ~(size_t)255;
    uint64_t* k0 = (uint64_t*)p;
    uint64_t* k1 = k0 + n;
    int32_t* v0 = (int32_t*)(k1 + n);
    int32_t* v1 = v0 + n;
    int32_t* cnt = v1 + n;
    uint32_t* found = (uint32_t*)(cnt + 256);
    cudaMemsetAsync(cnt, 0, sizeof(int32_t), st);
    cudaMemsetAsync(found, 0, 256 * sizeof(uint32_t), st);
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 4096);
    k_cretr_keys<<<grid, 256, 0, st>>>(D, S, s, since, want, k0, v0, cnt);
    cudaError_t e = cub::DeviceRadixSort::SortPairs(cub_tmp, tmp, k0, k1, v0, v1, (int)n, 0, 64, st);
    if (e != cudaSuccess) return (int)e;
    k_cretr_bump<<<grid, 256, 0, st>>>(D, S, s, now, v1, cnt, found);
    *sorted_out = v1, *cnt_out = cnt, *found_out = found;
    return (int)cudaGetLastError();
}
void launch_score_meta(const Cfg& C, const pikv_entry* m, const double* layers, int n_layers, int n, uint64_t now,
                       double* out, cudaStream_t st) {
    if (n > 0) k_score_meta<<<(n + 127) / 128, 128, 0, st>>>(C, m, layers, n_layers, n, now, out);
}
void launch_state_op(const Dims& D, const Cfg& C, const State& S, int s, int op, uint64_t a, uint64_t b,
                     const int32_t* experts, int n, double reward, cudaStream_t st) {
    k_state_op<<<1, 32, 0, st>>>(D, C, S, s, op, a, b, experts, n, reward);
}
void launch_read_heads(const Dims& D, const State& S, int s, const int64_t* slots, int n, float* kh, float* vh,
                       cudaStream_t st) {
    if (n > 0) k_read_heads<<<n, 256, 0, st>>>(D, S, s, slots, n, kh, vh);
}
void launch_head_mean(const float* w, int H, int n, float* out, cudaStream_t st) {
    if (n > 0) k_head_mean<<<(n + 255) / 256, 256, 0, st>>>(w, H, n, out);
}
void launch_codec_select(int decode, int codec, int64_t rows, int heads, int hd, int r, const int32_t* kept,
                         const float* x, float* y, cudaStream_t st) {
    const int64_t n = rows * heads * (decode ? hd : r);
    if (n > 0) k_codec_select<<<(unsigned)std::min<int64_t>((n + 255) / 256, 65535), 256, 0, st>>>(
        decode, codec, rows, heads, hd, r, kept, x, y);
}
void launch_col_var(const double* x, int n, int d, double* var, cudaStream_t st) {
    if (d > 0) k_col_var<<<(d + 127) / 128, 128, 0, st>>>(x, n, d, var);
}

}  // namespace pikv_dev
