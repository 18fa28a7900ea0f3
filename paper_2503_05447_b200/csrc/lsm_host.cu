// lsm_host.cu -- host orchestration of the LSM forward and of LSM sequence parallelism:
// argument validation with the reference's error texts, segment planning, workspace
// carving, TMA descriptors, launches, NCCL all-gather of the per-rank state payload.
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "common.h"
#include "internal.h"
#include "lsm_launch.h"

namespace lmoe_host {

// Optional per-phase timing (LMOE_FLAG_TIMING): CUDA events recorded on the caller's stream
// around each kernel; lmoe_timing_read() sums elapsed milliseconds per phase.
struct PhaseTimer {
    std::vector<cudaEvent_t> pool;
    std::vector<std::vector<cudaEvent_t>> pending;
    size_t next = 0;
    cudaEvent_t get() {
        if (next == pool.size()) {
            cudaEvent_t e;
            LMOE_CUDA_CHECK(cudaEventCreate(&e));
            pool.push_back(e);
        }
        return pool[next++];
    }
};
// Per calling thread (the library keeps no shared mutable state besides the launch counter):
// the timing events, the SP element accounting (RankGroup::comm_log, parallel.hpp:87-93) and
// the developer trace buffer belong to the thread that made the call.
static thread_local PhaseTimer g_timer;
static thread_local long long g_last_gather_elements = 0;
static thread_local unsigned long long* g_trace = nullptr;

static const char* kInstanceNames[] = {"bla",    "lightning", "retnet", "gla",   "deltanet",
                                       "gated_deltanet", "rebased", "gfw", "gateloop", "ttt",
                                       "titans", "s4",        "mamba",  "mamba2", "hgrn2",
                                       "rwkv6",  "rwkv7"};

const char* instance_name(int inst) {
    return (inst >= 0 && inst <= 16) ? kInstanceNames[inst] : "unknown";
}

// lmoe::decay_kind (lsm.hpp:64-85) restricted to what the device path implements.
int device_decay_mode(int inst) {
    switch (inst) {
        case LMOE_BLA: case LMOE_REBASED: return lmoe_dev::kDecayNone;
        case LMOE_LIGHTNING: case LMOE_RETNET: return lmoe_dev::kDecayConst;
        case LMOE_MAMBA2: return lmoe_dev::kDecayTokenScalar;
        case LMOE_GLA: case LMOE_HGRN2: case LMOE_RWKV6: return lmoe_dev::kDecayTokenVector;
        default: return -1;
    }
}

struct LsmPlan {
    int seg_len = 0, nseg = 0;
    // single-read forward (lsm_fused.cuh): fP CTAs per (b,h), fnseg segments of fseg_len
    int fP = 0, fseg_len = 0, fnseg = 0;
    size_t off_S = 0, off_z = 0, off_logD = 0, off_Min = 0, off_zin = 0, off_err = 0, off_ring = 0,
           off_flags = 0, off_ringD = 0, off_incl = 0, total = 0;
};

static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

// Single-read forward plan: P = floor(#SMs / (B*H)) CTAs per head (all co-resident), segments
// of c chunks, CTA j of a head taking segments j, j+P, ...  Cost per CTA ~ units x (c x
// (1 output step + ~0.3 state step) + ~1 per-unit hand-off / fill); c <= 8 keeps every CTA's
// K/V between its state and output reads in L2 (148 x 8 x 64 KB = 78 MB of 126 MB).
static void plan_fused(LsmPlan& pl, int B, int N, int H) {
    const int chunks = (N + lmoe_dev::kC - 1) / lmoe_dev::kC;
    const int BH = B * H;
    const int P = num_sms() / BH;
    if (P < 2 && chunks > 8) return;  // too many heads to split: the segment-parallel passes
    const int cmax = std::max(1, std::min(16, env_int("LMOE_FUSED_SEGC", 8)));
    double best = 1e300;
    for (int c = 1; c <= cmax; ++c) {
        const int units = (chunks + c - 1) / c;
        const int per_cta = (units + std::max(P, 1) - 1) / std::max(P, 1);
        const double cost = per_cta * (1.3 * c + 1.0);
        if (cost < best - 1e-9) {
            best = cost;
            pl.fseg_len = c * lmoe_dev::kC;
            pl.fnseg = units;
        }
    }
    pl.fP = std::max(1, std::min(P, pl.fnseg));
}

// Segment length: a multiple of the 128-token tile.  The B*H*nseg CTAs of the
// segment-parallel passes run one per SM; a pass costs about waves x (chunks per segment +
// a per-CTA fixed cost: prologue, pipeline fill and drain, ~2 chunks), so short slices
// (sequence parallelism) prefer one wave of longer segments over several waves of short ones.
static LsmPlan plan_lsm(int B, int N, int H, int D) {
    LsmPlan pl;
    const int C = lmoe_dev::kC;
    const int chunks = (N + C - 1) / C;
    const long long heads = (long long)B * H;
    const int sms = num_sms();
    constexpr double kFixedChunks = 2.0;
    double best = 1e300;
    for (int nseg = 1; nseg <= chunks; ++nseg) {
        const int seg_chunks = (chunks + nseg - 1) / nseg;
        if ((chunks + seg_chunks - 1) / seg_chunks != nseg) continue;  // same as a smaller nseg
        const long long w = (heads * nseg + sms - 1) / sms;
        const double cost = (double)w * (seg_chunks + kFixedChunks);
        if (cost < best - 1e-9) {
            best = cost;
            pl.seg_len = seg_chunks * C;
            pl.nseg = nseg;
        }
        if (w > 16) break;
    }
    const size_t heads_nseg = (size_t)heads * pl.nseg;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    pl.off_S = take(heads_nseg * D * D * 4);
    pl.off_z = take(heads_nseg * D * 4);
    pl.off_logD = take(heads_nseg * D * 4);  // per-row log decay for TokenVector kinds
    pl.off_Min = take(heads_nseg * D * D * 4);
    pl.off_zin = take(heads_nseg * D * 4);
    pl.off_err = take(64);
    plan_fused(pl, B, N, H);
    const size_t fR = 2 * (size_t)std::max(pl.fP, 1);
    pl.off_ring = take(heads * fR * D * D * 4);
    pl.off_flags = take(heads * fR * 4);
    pl.off_ringD = take(heads * fR * 4);
    pl.off_incl = take(heads * (size_t)std::max(pl.fP, 1) * D * D * 4);
    pl.total = off;
    return pl;
}

static void validate(const lmoe_lsm_desc* d, int B, int N, int H, int D, lmoe_dtype dt,
                     const void* q, const void* k, const void* v, const void* o) {
    if (!d) throw Error(LMOE_ERR_ARG, "lmoe_lsm_fwd: null descriptor");
    if (d->chunk_size < 1) throw Error(LMOE_ERR_ARG, "lsm_forward_chunked: chunk_size must be >= 1");
    if (D <= 0) throw Error(LMOE_ERR_ARG, "LsmSpec: nonpositive head dims");
    if (N < 1 || B < 1 || H < 1)
        throw Error(LMOE_ERR_ARG, "lsm_forward_sequential: need N >= 1 rows");
    if (d->use_normalizer) {
        // LsmSpec::validate (lsm.hpp:188-204)
        const int inst = d->instance;
        const bool diagonal = inst == LMOE_BLA || inst == LMOE_REBASED || inst == LMOE_LIGHTNING ||
                              inst == LMOE_RETNET || inst == LMOE_MAMBA2 || inst == LMOE_GLA ||
                              inst == LMOE_HGRN2 || inst == LMOE_RWKV6;
        if (!diagonal || inst == LMOE_HGRN2 || inst == LMOE_MAMBA2)
            throw Error(LMOE_ERR_ARG, std::string("LsmSpec: normalizer unsupported for instance ") +
                                          instance_name(inst));
    }
    if (device_decay_mode(d->instance) < 0)
        throw Error(LMOE_ERR_UNSUPPORTED,
                    std::string("lmoe_lsm_fwd: instance ") + instance_name(d->instance) +
                        " has no device kernel in this build");
    if (!((dt == LMOE_BF16 && D == 128) || (dt == LMOE_F32 && D == 64)))
        throw Error(LMOE_ERR_UNSUPPORTED,
                    "lmoe_lsm_fwd: supported (dtype, head_dim) pairs are (bf16, 128) and (f32, 64)");
    if (d->feature_map < 0 || d->feature_map > 2) throw Error(LMOE_ERR_ARG, "unknown feature map");
    if (!q || !k || !v || !o) throw Error(LMOE_ERR_ARG, "lmoe_lsm_fwd: null tensor");
}

// One LSM evaluation over a [B, N, H, D] view whose sequence stride is Nstride (>= N):
// the full tensor for lmoe_lsm_fwd, a rank slice for sequence parallelism.
struct LsmCall {
    const lmoe_lsm_desc* d;
    int B, N, Nstride, H, D;
    lmoe_dtype dt;
    const void *q, *k, *v;
    const float *b_pre, *a_raw;
    void* o;
    uint8_t* ws;
    LsmPlan pl;
    cudaStream_t st;
    const void* a_pre = nullptr;  // TokenVector gate pre-activations [B, N, H, D]
    std::vector<cudaEvent_t> ev;
    lmoe_dev::LsmFwdParams p{};
    lmoe_dev::LsmVariant var{};
    bool norm = false;
    bool vec = false;
    bool sp_local = false;  // SP phase A ran the local-state output pass (phase B corrects)
    int lw = 1;  // log-decay entries per state: 1, or D for TokenVector kinds
    int ld = 0;  // elements per token row of q, k, v, a_pre (0: H * D); o is always dense

    void mark() {
        if (!(d->flags & LMOE_FLAG_TIMING)) return;
        ev.push_back(g_timer.get());
        LMOE_CUDA_CHECK(cudaEventRecord(ev.back(), st));
    }
    void finish_timing() {
        if (!ev.empty()) g_timer.pending.push_back(ev);
        ev.clear();
    }

    void setup() {
        p.B = B; p.N = N; p.H = H; p.Nstride = Nstride;
        p.seg_len = pl.seg_len;
        p.nseg = pl.nseg;
        var.decay = device_decay_mode(d->instance);
        var.fm = d->feature_map;
        var.norm = d->use_normalizer ? 1 : 0;
        var.hgrn2 = d->instance == LMOE_HGRN2 ? 1 : 0;
        norm = var.norm != 0;
        vec = var.decay == lmoe_dev::kDecayTokenVector;
        lw = vec ? D : 1;
        if (vec && !a_pre) throw Error(LMOE_ERR_ARG, "lmoe_lsm_fwd: TokenVector instances need a_pre");
        p.log_a = var.decay == lmoe_dev::kDecayConst ? logf(d->scalar_decay) : 0.f;
        p.b_pre = b_pre;
        p.a_raw = a_raw;
        p.Sseg = reinterpret_cast<float*>(ws + pl.off_S);
        p.zseg = reinterpret_cast<float*>(ws + pl.off_z);
        p.logDseg = reinterpret_cast<float*>(ws + pl.off_logD);
        p.Min = reinterpret_cast<const float*>(ws + pl.off_Min);
        p.zin = reinterpret_cast<const float*>(ws + pl.off_zin);
        p.o = o;
        p.err = reinterpret_cast<int*>(ws + pl.off_err);
        p.fault = (d->flags & LMOE_FLAG_TEST_DECAY_FAULT) ? 1 : 0;
        // developer knobs: phase-3 schedule and a clock64 trace of CTA (0,0,0)
        static const int order = getenv("LMOE_OP_ORDER") ? atoi(getenv("LMOE_OP_ORDER")) : 1;
        p.order = order;
        p.trace = nullptr;
        if (getenv("LMOE_TRACE")) {
            if (!g_trace) {
                LMOE_CUDA_CHECK(cudaMalloc(&g_trace, (64 * 16 + 4 * 4096) * 8));
                LMOE_CUDA_CHECK(cudaMemset(g_trace, 0, (64 * 16 + 4 * 4096) * 8));
            }
            p.trace = g_trace;
        }
        if (var.decay == lmoe_dev::kDecayTokenScalar && (!b_pre || !a_raw))
            throw Error(LMOE_ERR_ARG, "lmoe_lsm_fwd: Mamba2 needs b_pre and a_raw");
    }

    template <typename T>
    CUtensorMap tmap(const void* base) const {
        using TT = lmoe_dev::TileTraits<T>;
        const CUtensorMapDataType tdt =
            sizeof(T) == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        const bool dense_out = base == o;
        return make_tmap_4d(base, tdt, sizeof(T), TT::D, H, N, B, TT::EPB, lmoe_dev::kC, Nstride,
                            dense_out ? 0 : ld);
    }

    template <typename T>
    void state_pass() {
        const CUtensorMap tk = tmap<T>(k), tv = tmap<T>(v);
        mark();
        const dim3 grid(pl.nseg, H, B);
        if (vec) {
            const CUtensorMap ta = tmap<T>(a_pre);
            if constexpr (sizeof(T) == 2)
                LMOE_CUDA_CHECK(lmoe_dev::launch_state_pass_vec_bf16(var, grid, st, tk, tv, ta, p));
            else
                LMOE_CUDA_CHECK(lmoe_dev::launch_state_pass_vec_f32(var, grid, st, tk, tv, ta, p));
        } else if constexpr (sizeof(T) == 2) {
            LMOE_CUDA_CHECK(lmoe_dev::launch_state_pass_bf16(var, grid, st, tk, tv, p));
        } else {
            LMOE_CUDA_CHECK(lmoe_dev::launch_state_pass_f32(var, grid, st, tk, tv, p));
        }
        ++g_launch_count;
    }
    // Segment prefix with carried-in state (M0, z0); writes per-segment M_in and the
    // inclusive total (Mfin/zfin with row stride fin_stride, and its total log decay).
    void combine(const float* M0, const float* z0, bool write_min, float* Mfin, float* zfin,
                 float* logDtot, int fin_stride, int rev = 0) {
        mark();
        const int nel = D * D + (norm ? D : 0);
        LMOE_CUDA_CHECK(lmoe_dev::launch_seg_combine(
            dim3((nel + 255) / 256, B * H), st, p.Sseg, p.zseg, p.logDseg, M0, z0,
            write_min ? const_cast<float*>(p.Min) : nullptr,
            write_min ? const_cast<float*>(p.zin) : nullptr, Mfin, zfin, logDtot, fin_stride,
            pl.nseg, D, D, norm ? 1 : 0, lw, rev, p.err));
        ++g_launch_count;
    }
    template <typename T>
    void output_pass() {
        const CUtensorMap tq = tmap<T>(q), tk = tmap<T>(k), tv = tmap<T>(v), to = tmap<T>(o);
        mark();
        const dim3 grid(pl.nseg, H, B);
        if (vec) {
            const CUtensorMap ta = tmap<T>(a_pre);
            if constexpr (sizeof(T) == 2)
                LMOE_CUDA_CHECK(lmoe_dev::launch_output_pass_vec_bf16(var, grid, st, tq, tk, tv, ta, to, p));
            else
                LMOE_CUDA_CHECK(lmoe_dev::launch_output_pass_vec_f32(var, grid, st, tq, tk, tv, ta, to, p));
        } else if constexpr (sizeof(T) == 2) {
            LMOE_CUDA_CHECK(lmoe_dev::launch_output_pass_bf16(var, grid, st, tq, tk, tv, to, p));
        } else {
            LMOE_CUDA_CHECK(lmoe_dev::launch_output_pass_f32(var, grid, st, tq, tk, tv, to, p));
        }
        ++g_launch_count;
        mark();
    }
    // the single-read forward applies to bf16 / D = 128 scalar-decay kinds without normaliser
    // (forward order, no backward side channel).  It is opt-in (LMOE_FUSED=1): measured at
    // config 3 it runs 2.8 ms against the three passes' 1.19 ms, bound by the segment-to-
    // segment hand-off (~10 us per hop, 256 hops per head) and by its state steps not
    // overlapping its output steps.
    bool fused_ok() const {
        return env_int("LMOE_FUSED", 0) != 0 && dt == LMOE_BF16 && D == 128 && !norm && !vec && var.rev == 0 &&
               p.mst == nullptr && !p.out_f32 && !p.nomask && pl.fP >= 1;
    }
    void fused(const float* M0, float* M_out) {
        using bf = __nv_bfloat16;
        const CUtensorMap tq = tmap<bf>(q), tk = tmap<bf>(k), tv = tmap<bf>(v), to = tmap<bf>(o);
        lmoe_dev::LsmFwdParams fp = p;
        fp.seg_len = pl.fseg_len;
        fp.nseg = pl.fnseg;
        fp.fP = pl.fP;
        fp.fR = 2 * pl.fP;
        fp.ring = reinterpret_cast<float*>(ws + pl.off_ring);
        fp.flags = reinterpret_cast<int*>(ws + pl.off_flags);
        fp.ringD = reinterpret_cast<float*>(ws + pl.off_ringD);
        fp.incl = reinterpret_cast<float*>(ws + pl.off_incl);
        fp.Min = M0;
        fp.Mfin = M_out;
        fp.order = env_int("LMOE_FUSED_HINT", 1);
        fp.fdbg = getenv("LMOE_FUSED_DEBUG_PTR") ? reinterpret_cast<float*>(strtoull(getenv("LMOE_FUSED_DEBUG_PTR"), nullptr, 10)) : nullptr;
        LMOE_CUDA_CHECK(cudaMemsetAsync(fp.flags, 0, (size_t)B * H * fp.fR * 4, st));
        mark();
        LMOE_CUDA_CHECK(lmoe_dev::launch_fused_fwd_bf16(var, pl.fP * B * H, st, tq, tk, tv, to, fp));
        ++g_launch_count;
        mark();
    }
    // Local-state forward (decaying scalar kinds): the output pass runs every segment but the
    // first from a zero state and writes each segment's final state; the combine turns those
    // into the entering states; lsm_local_fix adds (q e^{Gseg}) M_in to the first chunks of each
    // segment, until the decay from the segment start leaves the fp32 range.  No state pass: the
    // step reads q, k, v once plus the corrected chunks' q and o.  For a constant decay the
    // corrected span is known: taken when it costs less than the state pass it replaces.
    bool local_ok() const {
        if (env_int("LMOE_LOCAL", 1) == 0 || fused_ok()) return false;
        if (!(dt == LMOE_BF16 && D == 128 && !norm && var.rev == 0 && var.fm == 0 && p.mst == nullptr &&
              !p.out_f32 && !p.nomask))
            return false;
        if (vec) return env_int("LMOE_LOCAL_VEC", 1) != 0;  // lsm_local_fix_vec
        if (var.decay == lmoe_dev::kDecayTokenScalar) return true;
        if (var.decay != lmoe_dev::kDecayConst || !(p.log_a < 0.f)) return false;
        const double span_tokens = 88.0 / -(double)p.log_a;  // tokens until e^{G} < e^{-88}
        const double fix_bytes = 768.0 * std::min<double>(span_tokens + lmoe_dev::kC, pl.seg_len) * (pl.nseg - 1);
        return fix_bytes < 0.8 * 512.0 * N;
    }
    void local_pass(const float* M0, float* M_out) {
        using bf = __nv_bfloat16;
        // every segment from a zero state (segment states are then the combine's inputs); with
        // an initial state segment 0 is corrected too (its entering state M0)
        p.local = 1;
        p.Mloc0 = nullptr;
        output_pass<bf>();  // timing phase 0
        p.local = 0;
        combine(M0, nullptr, true, M_out, nullptr, nullptr, 0);  // phase 2
        mark();
        local_fix(M0 ? pl.nseg : pl.nseg - 1);  // phase 3: the correction
        mark();
    }
    // correct the last nfix segments' first chunks with the entering states in p.Min
    void local_fix(int nfix) {
        using bf = __nv_bfloat16;
        if (nfix <= 0) return;
        const CUtensorMap tq = tmap<bf>(q), to = tmap<bf>(o);
        if (vec) {
            const CUtensorMap ta = tmap<bf>(a_pre);
            LMOE_CUDA_CHECK(lmoe_dev::launch_local_fix_vec_bf16(dim3(nfix, H, B), st, tq, ta, to, p));
        } else {
            LMOE_CUDA_CHECK(lmoe_dev::launch_local_fix_bf16(var.decay, dim3(nfix, H, B), st, tq, to, p));
        }
        ++g_launch_count;
    }
    void clear_err() { LMOE_CUDA_CHECK(cudaMemsetAsync(p.err, 0, 64, st)); }
    void check_err() {
        if (!(d->flags & LMOE_FLAG_CHECK)) return;
        int err[3] = {0, 0, 0};
        LMOE_CUDA_CHECK(cudaMemcpyAsync(err, p.err, sizeof(err), cudaMemcpyDeviceToHost, st));
        LMOE_CUDA_CHECK(cudaStreamSynchronize(st));
        if (err[2])  // TokenVector chunk whose half-chunk decay span leaves the fp32 range
            throw Error(LMOE_ERR_NONFINITE, "non-finite output in div");
        if (err[0])
            throw Error(LMOE_ERR_DEGENERATE,
                        std::string("degenerate normalizer in instance ") + instance_name(d->instance));
        if (err[1])
            throw Error(LMOE_ERR_NONFINITE,
                        std::string("non-finite memory state in instance ") + instance_name(d->instance));
    }
};

template <typename T>
static void run_local(LsmCall& c, const float* M0, const float* z0, float* M_out, float* z_out) {
    c.setup();
    c.clear_err();
    if (c.fused_ok()) {
        c.fused(M0, M_out);
    } else if (c.local_ok() && z0 == nullptr && z_out == nullptr) {
        c.local_pass(M0, M_out);
    } else {
        c.state_pass<T>();
        c.combine(M0, z0, true, M_out, z_out, nullptr, 0);
        c.output_pass<T>();
    }
    c.finish_timing();
    c.check_err();
}

// [M | z? | log D]: log D is a scalar, or a d_k vector for TokenVector kinds
static int payload_lw(const lmoe_lsm_desc* d, int D) {
    return device_decay_mode(d->instance) == lmoe_dev::kDecayTokenVector ? D : 1;
}
static size_t payload_floats(const lmoe_lsm_desc* d, int D) {
    return (size_t)D * D + (d->use_normalizer ? D : 0) + payload_lw(d, D);
}

struct SpWorkspace {
    LsmPlan pl;
    size_t region = 0;  // bytes of the per-slice LSM region (max over the slice lengths served)
    size_t off_payload = 0, off_gathered = 0, off_M0 = 0, off_z0 = 0, off_err = 0, total = 0;
};

// n_min: the shortest slice this workspace serves (loopback: N / world, while N_local is the
// longest).  plan_lsm is not monotone in N, so the per-slice region is the max over both
// lengths; every slice carves its own plan inside [0, region) and shares one error slot.
static SpWorkspace plan_sp(const lmoe_lsm_desc* d, int B, int N_local, int H, int D, int world,
                           int n_min = -1) {
    SpWorkspace w;
    w.pl = plan_lsm(B, N_local, H, D);
    w.region = w.pl.total;
    if (n_min > 0 && n_min != N_local) w.region = std::max(w.region, plan_lsm(B, n_min, H, D).total);
    const size_t BH = (size_t)B * H, P = payload_floats(d, D);
    size_t off = align_up(w.region, 256);
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    w.off_payload = take(BH * P * 4);
    w.off_gathered = take((size_t)world * BH * P * 4);
    w.off_M0 = take(BH * D * D * 4);
    w.off_z0 = take(BH * D * 4);
    w.off_err = take(64);
    w.total = off;
    return w;
}

// Phase A of sp_lsm_masked_rank (parallel.hpp:313-327): local state from zero and the
// payload [M | z? | log D] per (b,h), written to `payload`.
template <typename T>
static void sp_phase_a(LsmCall& c, float* payload) {
    const int P = (int)payload_floats(c.d, c.D);
    if constexpr (sizeof(T) == 2) {
        if (c.o != nullptr && c.local_ok()) {  // local-state forward: the output pass first, from zero
                                               // states (payload-only callers, o == NULL, skip it)
            c.sp_local = true;
            c.p.local = 1;
            c.p.Mloc0 = nullptr;
            c.output_pass<T>();
            c.p.local = 0;
            c.combine(nullptr, nullptr, false, payload, nullptr, payload + P - c.lw, P);
            return;
        }
    }
    c.state_pass<T>();
    c.combine(nullptr, nullptr, false, payload, c.norm ? payload + c.D * c.D : nullptr,
              payload + P - c.lw, P);
}
// Phase B (parallel.hpp:340-373): decayed exclusive prefix over ranks < rank, then the
// output pass with the carried-in state.
template <typename T>
static void sp_phase_b(LsmCall& c, const float* gathered, int rank, float* M0, float* z0,
                       float* M_out, float* z_out) {
    const int P = (int)payload_floats(c.d, c.D);
    (void)M0; (void)z0;
    c.mark();  // rank-combine phase (fused with the segment combine below)
    c.mark();
    LMOE_CUDA_CHECK(lmoe_dev::launch_rank_seg_combine(gathered, P, c.B * c.H, rank, c.p.Sseg, c.p.zseg, c.p.logDseg,
                                                      const_cast<float*>(c.p.Min), const_cast<float*>(c.p.zin),
                                                      M_out, z_out, c.pl.nseg, c.D, c.D, c.norm ? 1 : 0, c.lw,
                                                      c.st));
    ++g_launch_count;
    if (c.sp_local) {  // the entering states are known now: correct each segment's first chunks
        c.mark();
        c.local_fix(rank > 0 ? c.pl.nseg : c.pl.nseg - 1);  // rank 0 carries nothing into segment 0
        c.mark();
        return;
    }
    c.output_pass<T>();
}

#define NCCL_CHECK(x)                                                                      \
    do {                                                                                   \
        ncclResult_t r_ = (x);                                                             \
        if (r_ != ncclSuccess)                                                             \
            throw Error(LMOE_ERR_NCCL, std::string("NCCL error: ") + ncclGetErrorString(r_)); \
    } while (0)

}  // namespace lmoe_host

using namespace lmoe_host;

extern "C" size_t lmoe_lsm_fwd_workspace_size(const lmoe_lsm_desc* desc, int B, int N, int H,
                                              int D, lmoe_dtype dtype) {
    (void)desc; (void)dtype;
    if (B < 1 || N < 1 || H < 1 || D < 1) return 0;
    return plan_lsm(B, N, H, D).total;
}

extern "C" int lmoe_lsm_fwd_plan(const lmoe_lsm_desc* desc, int B, int N, int H, int D, lmoe_dtype dtype,
                                 int* info) {
    return guarded([&]() {
        if (!desc || !info || B < 1 || N < 1 || H < 1 || D < 1) throw Error(LMOE_ERR_ARG, "lmoe_lsm_fwd_plan: bad arguments");
        const LsmPlan pl = plan_lsm(B, N, H, D);
        LsmCall c{desc, B, N, N, H, D, dtype, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, pl,
                  nullptr, nullptr};
        c.var.decay = device_decay_mode(desc->instance);
        c.var.fm = desc->feature_map;
        c.norm = desc->use_normalizer != 0;
        c.vec = c.var.decay == lmoe_dev::kDecayTokenVector;
        c.p.log_a = c.var.decay == lmoe_dev::kDecayConst ? logf(desc->scalar_decay) : 0.f;
        const bool f = c.var.decay >= 0 && c.fused_ok();
        const bool loc = !f && c.var.decay >= 0 && c.local_ok();
        info[0] = f ? 1 : (loc ? 2 : 0);
        info[1] = f ? pl.fnseg : pl.nseg;
        info[2] = f ? pl.fseg_len : pl.seg_len;
        info[3] = f ? pl.fP : pl.nseg;
    });
}

extern "C" int lmoe_lsm_fwd_num_launches(const lmoe_lsm_desc* desc) {
    (void)desc;
    return 3;
}

// Sums per-phase device milliseconds over all LMOE_FLAG_TIMING calls since the last read.
extern "C" int lmoe_timing_read(float* ms_out, int nphase) {
    int calls = 0;
    int rc = guarded([&]() {
        for (int i = 0; i < nphase; ++i) ms_out[i] = 0.f;
        for (auto& ev : g_timer.pending) {
            LMOE_CUDA_CHECK(cudaEventSynchronize(ev.back()));
            for (size_t i = 0; i + 1 < ev.size() && (int)i < nphase; ++i) {
                float ms = 0.f;
                LMOE_CUDA_CHECK(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
                ms_out[i] += ms;
            }
            ++calls;
        }
        g_timer.pending.clear();
        g_timer.next = 0;
    });
    return rc == LMOE_OK ? calls : -rc;
}

extern "C" int lmoe_lsm_fwd(const lmoe_lsm_desc* desc, int B, int N, int H, int D,
                            lmoe_dtype dtype, const void* q, const void* k, const void* v,
                            const void* a_pre, const float* b_pre, const float* a_raw,
                            const float* M0, const float* z0, void* o, float* M_out,
                            float* z_out, void* workspace, size_t workspace_bytes,
                            lmoe_stream_t stream) {
    return guarded([&]() {
        validate(desc, B, N, H, D, dtype, q, k, v, o);
        LsmCall c{desc, B, N, N, H, D, dtype, q, k, v, b_pre, a_raw, o,
                  static_cast<uint8_t*>(workspace), plan_lsm(B, N, H, D),
                  reinterpret_cast<cudaStream_t>(stream), a_pre};
        if (!workspace || workspace_bytes < c.pl.total)
            throw Error(LMOE_ERR_ARG, "lmoe_lsm_fwd: workspace too small (need " +
                                          std::to_string(c.pl.total) + " bytes)");
        if (dtype == LMOE_BF16) run_local<__nv_bfloat16>(c, M0, z0, M_out, z_out);
        else run_local<float>(c, M0, z0, M_out, z_out);
    });
}

// ------------------------------------------------------------------ sequence parallelism
extern "C" size_t lmoe_sp_payload_floats(const lmoe_lsm_desc* desc, int B, int H, int D) {
    return (size_t)B * H * payload_floats(desc, D);
}

extern "C" size_t lmoe_sp_lsm_fwd_workspace_size(const lmoe_lsm_desc* desc, int B, int N_local,
                                                 int H, int D, lmoe_dtype dtype, int world) {
    (void)dtype;
    if (!desc || B < 1 || N_local < 1 || H < 1 || D < 1 || world < 1) return 0;
    return plan_sp(desc, B, N_local, H, D, world).total;
}

extern "C" long long lmoe_sp_last_gather_elements(void) { return g_last_gather_elements; }

extern "C" int lmoe_nccl_unique_id(void* id128) {
    return guarded([&]() {
        ncclUniqueId id;
        NCCL_CHECK(ncclGetUniqueId(&id));
        static_assert(sizeof(id) == 128, "ncclUniqueId size");
        memcpy(id128, &id, sizeof(id));
    });
}

extern "C" int lmoe_nccl_comm_init(void** comm, int world, int rank, const void* id128) {
    return guarded([&]() {
        ncclUniqueId id;
        memcpy(&id, id128, sizeof(id));
        ncclComm_t c;
        NCCL_CHECK(ncclCommInitRank(&c, world, id, rank));
        *comm = c;
    });
}

extern "C" int lmoe_nccl_comm_destroy(void* comm) {
    return guarded([&]() { NCCL_CHECK(ncclCommDestroy(static_cast<ncclComm_t>(comm))); });
}

namespace lmoe_host {
size_t lsm_mixer_ws(const lmoe_lsm_desc* d, int B, int N, int H, int D, int world) {
    return plan_sp(d, B, N, H, D, world).total;
}

void lsm_mixer_core(const lmoe_lsm_desc* desc, int B, int N_local, int H, int D, lmoe_dtype dtype,
                    const void* q, const void* k, const void* v, const void* a_pre, int ld, const float* b_pre,
                    const float* a_raw, void* o, void* nccl_comm, int rank, int world, void* workspace,
                    size_t workspace_bytes, cudaStream_t st, float* M_out, float* z_out) {
    validate(desc, B, N_local, H, D, dtype, q, k, v, o);
    if (world < 1 || rank < 0 || rank >= world) throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_fwd: bad rank");
    if (world > 1 && !nccl_comm) throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_fwd: null communicator");
    const SpWorkspace w = plan_sp(desc, B, N_local, H, D, world);
    if (!workspace || workspace_bytes < w.total)
        throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_fwd: workspace too small (need " +
                                      std::to_string(w.total) + " bytes)");
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    LsmCall c{desc, B, N_local, N_local, H, D, dtype, q, k, v, b_pre, a_raw, o, ws, w.pl, st, a_pre};
    c.ld = ld;
    c.setup();
    c.clear_err();
    float* payload = reinterpret_cast<float*>(ws + w.off_payload);
    float* gathered = reinterpret_cast<float*>(ws + w.off_gathered);
    float* M0 = reinterpret_cast<float*>(ws + w.off_M0);
    float* z0 = reinterpret_cast<float*>(ws + w.off_z0);
    const size_t P = (size_t)B * H * payload_floats(desc, D);
    g_last_gather_elements = (long long)world * (long long)P;
    // developer knob (tools/sp_scaling_probe.py): run the multi-rank phase structure at world 1,
    // a device copy standing in for the all-gather
    const bool force_sp = getenv("LMOE_SP_FORCE") != nullptr;
    if (world == 1 && !force_sp && !nccl_comm) {
        // a gather over one rank is the identity and rank 0 carries nothing in: the local
        // pass (state pass, segment prefix, output pass); the empty marks keep the phase
        // timers' layout (all-gather, rank combine).  With a (1-rank) communicator the SP
        // structure runs instead, ncclAllGather included.
        if (c.fused_ok()) {  // one single-read launch (timing phase 0)
            c.fused(nullptr, M_out);
            c.finish_timing();
            c.check_err();
            return;
        }
        if (c.local_ok() && z_out == nullptr) {  // local-state forward (phases: output, -, combine, fix)
            c.local_pass(nullptr, M_out);
            c.finish_timing();
            c.check_err();
            return;
        }
        if (dtype == LMOE_BF16) c.state_pass<__nv_bfloat16>();
        else c.state_pass<float>();
        c.combine(nullptr, nullptr, true, M_out, z_out, nullptr, 0);
        c.mark();
        c.mark();
        c.mark();
        if (dtype == LMOE_BF16) c.output_pass<__nv_bfloat16>();
        else c.output_pass<float>();
        c.finish_timing();
        c.check_err();
        return;
    }
    if (dtype == LMOE_BF16) sp_phase_a<__nv_bfloat16>(c, payload);
    else sp_phase_a<float>(c, payload);
    c.mark();
    if (nccl_comm)
        NCCL_CHECK(ncclAllGather(payload, gathered, P, ncclFloat, static_cast<ncclComm_t>(nccl_comm), st));
    else
        LMOE_CUDA_CHECK(cudaMemcpyAsync(gathered, payload, P * 4, cudaMemcpyDeviceToDevice, st));
    if (dtype == LMOE_BF16) sp_phase_b<__nv_bfloat16>(c, gathered, rank, M0, z0, M_out, z_out);
    else sp_phase_b<float>(c, gathered, rank, M0, z0, M_out, z_out);
    c.finish_timing();
    c.check_err();
}

void lsm_mixer_core(const lmoe_lsm_desc* d, int B, int N, int H, int D, lmoe_dtype dt, const void* q,
                    const void* k, const void* v, const void* a_pre, int ld, const float* b_pre,
                    const float* a_raw, void* o, void* comm, int rank, int world, void* ws, size_t ws_bytes,
                    cudaStream_t st) {
    lsm_mixer_core(d, B, N, H, D, dt, q, k, v, a_pre, ld, b_pre, a_raw, o, comm, rank, world, ws, ws_bytes, st,
                   nullptr, nullptr);
}
}  // namespace lmoe_host

// sp_lsm_masked_rank (parallel.hpp:303-376) for this rank's contiguous slice
// (chunk_range, parallel.hpp:192-197): local pass, ONE ncclAllGather of the all-heads
// payload, decayed prefix over earlier ranks, output pass.
extern "C" int lmoe_sp_lsm_fwd(const lmoe_lsm_desc* desc, int B, int N_local, int H, int D,
                               lmoe_dtype dtype, const void* q, const void* k, const void* v,
                               const void* a_pre, const float* b_pre, const float* a_raw,
                               void* o, float* M_out, float* z_out, void* nccl_comm, int rank,
                               int world, void* workspace, size_t workspace_bytes,
                               lmoe_stream_t stream) {
    return guarded([&]() {
        lsm_mixer_core(desc, B, N_local, H, D, dtype, q, k, v, a_pre, 0, b_pre, a_raw, o, nccl_comm, rank, world,
                       workspace, workspace_bytes, reinterpret_cast<cudaStream_t>(stream), M_out, z_out);
    });
}

// The same algorithm with `world` virtual ranks on this device over the full [B,N,H,D]
// sequence: the all-gather is a device copy of each rank's payload into its slot.
extern "C" size_t lmoe_sp_lsm_fwd_loopback_workspace_size(const lmoe_lsm_desc* desc, int B, int N,
                                                          int H, int D, lmoe_dtype dtype, int world) {
    (void)dtype;
    if (!desc || world < 1 || N < world) return 0;
    return plan_sp(desc, B, (N + world - 1) / world, H, D, world, N / world).total;
}

extern "C" int lmoe_sp_lsm_fwd_loopback(const lmoe_lsm_desc* desc, int B, int N, int H, int D,
                                        lmoe_dtype dtype, const void* q, const void* k,
                                        const void* v, const void* a_pre, const float* b_pre,
                                        const float* a_raw, void* o, float* M_out, float* z_out,
                                        int world, void* workspace, size_t workspace_bytes,
                                        lmoe_stream_t stream) {
    return guarded([&]() {
        validate(desc, B, N, H, D, dtype, q, k, v, o);
        (void)a_pre;
        if (world < 1 || N < world) throw Error(LMOE_ERR_ARG, "chunk_range: need at least one row per rank");
        const SpWorkspace w = plan_sp(desc, B, (N + world - 1) / world, H, D, world, N / world);
        if (!workspace || workspace_bytes < w.total)
            throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_fwd_loopback: workspace too small");
        uint8_t* ws = static_cast<uint8_t*>(workspace);
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const size_t esz = dtype == LMOE_BF16 ? 2 : 4;
        const size_t P = (size_t)B * H * payload_floats(desc, D);
        float* gathered = reinterpret_cast<float*>(ws + w.off_gathered);
        float* M0 = reinterpret_cast<float*>(ws + w.off_M0);
        float* z0 = reinterpret_cast<float*>(ws + w.off_z0);
        auto slice_call = [&](int r) {
            const int base = N / world, rem = N % world;  // chunk_range (parallel.hpp:192-197)
            const int r0 = r * base + std::min(r, rem);
            const int len = base + (r < rem ? 1 : 0);
            const size_t off = (size_t)r0 * H * D * esz;
            LsmCall c{desc, B, len, N, H, D, dtype,
                      static_cast<const uint8_t*>(q) + off, static_cast<const uint8_t*>(k) + off,
                      static_cast<const uint8_t*>(v) + off, b_pre ? b_pre + (size_t)r0 * H : nullptr,
                      a_raw, static_cast<uint8_t*>(o) + off, ws, plan_lsm(B, len, H, D), st,
                      a_pre ? static_cast<const uint8_t*>(a_pre) + off : nullptr};
            c.setup();
            c.p.err = reinterpret_cast<int*>(ws + w.off_err);  // one error slot for all slices
            return c;
        };
        slice_call(0).clear_err();
        for (int r = 0; r < world; ++r) {
            LsmCall c = slice_call(r);
            if (dtype == LMOE_BF16) sp_phase_a<__nv_bfloat16>(c, gathered + r * P);
            else sp_phase_a<float>(c, gathered + r * P);
        }
        g_last_gather_elements = (long long)world * (long long)P;
        for (int r = 0; r < world; ++r) {
            LsmCall c = slice_call(r);
            const bool last = r == world - 1;
            if (dtype == LMOE_BF16) {
                // the slices share the segment-state region: recompute this slice's states; in the
                // local-state mode phase A already wrote its output from zero states
                c.state_pass<__nv_bfloat16>();
                c.sp_local = c.local_ok();
                sp_phase_b<__nv_bfloat16>(c, gathered, r, M0, z0, last ? M_out : nullptr, last ? z_out : nullptr);
            } else {
                c.state_pass<float>();
                sp_phase_b<float>(c, gathered, r, M0, z0, last ? M_out : nullptr, last ? z_out : nullptr);
            }
            if (last) c.check_err();
        }
    });
}

// ------------------------------------------------------------------ unmasked SP (Alg. 1)
// sp_lsm_nomask_rank (parallel.hpp:282-297): local phiK^T V, ONE all-gather of the
// T * d_k * d_v state elements per head, global sum, O = phiQ . sum.
namespace lmoe_host {
static void validate_nomask(const lmoe_lsm_desc* d) {
    if (device_decay_mode(d->instance) != lmoe_dev::kDecayNone)
        throw Error(LMOE_ERR_ARG, "sp_forward_nomask: requires an undecayed instance");
    if (d->use_normalizer) throw Error(LMOE_ERR_ARG, "sp_forward_nomask: normalizer unsupported");
}
template <typename T>
static void nomask_local_state(LsmCall& c, float* slot) {
    c.state_pass<T>();
    c.combine(nullptr, nullptr, false, slot, nullptr, nullptr, c.D * c.D);
}
template <typename T>
static void nomask_output(LsmCall& c, const float* Mglobal) {
    c.p.Min = Mglobal;
    c.p.nomask = 1;
    c.output_pass<T>();
}
}  // namespace lmoe_host

extern "C" size_t lmoe_sp_lsm_nomask_workspace_size(const lmoe_lsm_desc* desc, int B, int N_local, int H,
                                                    int D, lmoe_dtype dtype, int world) {
    return lmoe_sp_lsm_fwd_workspace_size(desc, B, N_local, H, D, dtype, world);
}

extern "C" int lmoe_sp_lsm_nomask_fwd(const lmoe_lsm_desc* desc, int B, int N_local, int H, int D,
                                      lmoe_dtype dtype, const void* q, const void* k, const void* v,
                                      void* o, void* nccl_comm, int rank, int world, void* workspace,
                                      size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        validate(desc, B, N_local, H, D, dtype, q, k, v, o);
        validate_nomask(desc);
        if (world < 1 || rank < 0 || rank >= world) throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_nomask_fwd: bad rank");
        if (world > 1 && !nccl_comm) throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_nomask_fwd: null communicator");
        const SpWorkspace w = plan_sp(desc, B, N_local, H, D, world);
        if (!workspace || workspace_bytes < w.total)
            throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_nomask_fwd: workspace too small (need " +
                                          std::to_string(w.total) + " bytes)");
        uint8_t* ws = static_cast<uint8_t*>(workspace);
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        LsmCall c{desc, B, N_local, N_local, H, D, dtype, q, k, v, nullptr, nullptr, o, ws, w.pl, st, nullptr};
        c.setup();
        c.clear_err();
        float* payload = reinterpret_cast<float*>(ws + w.off_payload);
        float* gathered = reinterpret_cast<float*>(ws + w.off_gathered);
        float* Mg = reinterpret_cast<float*>(ws + w.off_M0);
        const size_t P = (size_t)B * H * D * D;
        if (dtype == LMOE_BF16) nomask_local_state<__nv_bfloat16>(c, payload);
        else nomask_local_state<float>(c, payload);
        if (nccl_comm) {
            NCCL_CHECK(ncclAllGather(payload, gathered, P, ncclFloat, static_cast<ncclComm_t>(nccl_comm), st));
        } else {
            LMOE_CUDA_CHECK(cudaMemcpyAsync(gathered, payload, P * 4, cudaMemcpyDeviceToDevice, st));
        }
        g_last_gather_elements = (long long)world * (long long)P;
        LMOE_CUDA_CHECK(lmoe_dev::launch_sum_states(gathered, world, B * H, D * D, Mg, st));
        ++g_launch_count;
        if (dtype == LMOE_BF16) nomask_output<__nv_bfloat16>(c, Mg);
        else nomask_output<float>(c, Mg);
        c.finish_timing();
        c.check_err();
    });
}

extern "C" int lmoe_sp_lsm_nomask_fwd_loopback(const lmoe_lsm_desc* desc, int B, int N, int H, int D,
                                               lmoe_dtype dtype, const void* q, const void* k, const void* v,
                                               void* o, int world, void* workspace, size_t workspace_bytes,
                                               lmoe_stream_t stream) {
    return guarded([&]() {
        validate(desc, B, N, H, D, dtype, q, k, v, o);
        validate_nomask(desc);
        if (world < 1 || N < world) throw Error(LMOE_ERR_ARG, "chunk_range: need at least one row per rank");
        const SpWorkspace w = plan_sp(desc, B, (N + world - 1) / world, H, D, world, N / world);
        if (!workspace || workspace_bytes < w.total)
            throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_nomask_fwd_loopback: workspace too small");
        uint8_t* ws = static_cast<uint8_t*>(workspace);
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const size_t esz = dtype == LMOE_BF16 ? 2 : 4;
        const size_t P = (size_t)B * H * D * D;
        float* gathered = reinterpret_cast<float*>(ws + w.off_gathered);
        float* Mg = reinterpret_cast<float*>(ws + w.off_M0);
        auto slice_call = [&](int r) {
            const int base = N / world, rem = N % world;  // chunk_range (parallel.hpp:192-197)
            const int r0 = r * base + std::min(r, rem);
            const int len = base + (r < rem ? 1 : 0);
            const size_t off = (size_t)r0 * H * D * esz;
            LsmCall c{desc, B, len, N, H, D, dtype,
                      static_cast<const uint8_t*>(q) + off, static_cast<const uint8_t*>(k) + off,
                      static_cast<const uint8_t*>(v) + off, nullptr, nullptr,
                      static_cast<uint8_t*>(o) + off, ws, plan_lsm(B, len, H, D), st, nullptr};
            c.setup();
            c.p.err = reinterpret_cast<int*>(ws + w.off_err);
            return c;
        };
        slice_call(0).clear_err();
        for (int r = 0; r < world; ++r) {
            LsmCall c = slice_call(r);
            if (dtype == LMOE_BF16) nomask_local_state<__nv_bfloat16>(c, gathered + r * P);
            else nomask_local_state<float>(c, gathered + r * P);
        }
        g_last_gather_elements = (long long)world * (long long)P;
        LMOE_CUDA_CHECK(lmoe_dev::launch_sum_states(gathered, world, B * H, D * D, Mg, st));
        ++g_launch_count;
        for (int r = 0; r < world; ++r) {
            LsmCall c = slice_call(r);
            if (dtype == LMOE_BF16) nomask_output<__nv_bfloat16>(c, Mg);
            else nomask_output<float>(c, Mg);
        }
        slice_call(0).check_err();
    });
}

// ------------------------------------------------------------------------------- backward
// Three chunk passes, each a segment-parallel state pass + combine + output pass:
//   dq pass  (forward order)  q'=dO, k'=v, v'=phi(k), M0' = M0^T    -> dphi(q) fp32, M_N^T
//   dk pass  (REV)            q'=v,  k'=dO, v'=phi(q), dM' = dM_f^T -> dkeff fp32
//   dv pass  (REV)            q'=keff, k'=phi(q), v'=dO, dM = dM_f  -> dv, dM0
// then the chain rule (lsm_bwd_kernels.cu) and the Mamba2 gate gradients from the per-chunk
// state snapshots of the dq / dk passes (lsm_dgate.cu).
namespace lmoe_host {
struct BwdPlan {
    LsmPlan pl;
    size_t off_dphq = 0, off_dkef = 0, off_phq = 0, off_phk = 0, off_M0T = 0, off_dMfT = 0,
           off_MfinT = 0, off_dkfin = 0, off_dkf = 0, off_mst = 0, off_dmst = 0, off_bd = 0, total = 0;
};
static BwdPlan plan_bwd(const lmoe_lsm_desc* d, int B, int N, int H, int D, lmoe_dtype dt) {
    BwdPlan w;
    w.pl = plan_lsm(B, N, H, D);
    const size_t act = (size_t)B * N * H * D, esz = dt == LMOE_BF16 ? 2 : 4;
    const size_t BH = (size_t)B * H;
    size_t off = align_up(w.pl.total, 256);
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    w.off_dphq = take(act * 4);
    w.off_dkef = take(act * 4);
    if (d && d->feature_map != 0) {
        w.off_phq = take(act * esz);
        w.off_phk = take(act * esz);
    }
    w.off_M0T = take(BH * D * D * 4);
    w.off_dMfT = take(BH * D * D * 4);
    w.off_MfinT = take(BH * D * D * 4);
    w.off_dkfin = take(BH * D * D * 4);
    w.off_dkf = take(BH * N * 4);
    const size_t nchunk = (N + lmoe_dev::kC - 1) / lmoe_dev::kC;
    if (d && device_decay_mode(d->instance) == lmoe_dev::kDecayTokenScalar) {
        w.off_mst = take(BH * nchunk * D * D * esz);
        w.off_dmst = take(BH * nchunk * D * D * esz);
    }
    if (d && device_decay_mode(d->instance) == lmoe_dev::kDecayTokenVector) {
        // chunk-boundary states and adjoints (bf16) and their row dots, lsm_vec_bwd.cu
        w.off_mst = take(BH * (nchunk + 1) * D * D * 2);
        w.off_dmst = take(BH * (nchunk + 1) * D * D * 2);
        w.off_bd = take(BH * (nchunk + 1) * D * 4);
    }
    w.total = off;
    return w;
}

// TokenVector (GLA / HGRN2 / RWKV6) backward, bf16 / D = 128: chunk-boundary states and
// adjoints by two carry passes, then one fully parallel fused kernel per chunk
// (lsm_vec_bwd.cu).  q / k are the feature-mapped inputs; dq / dk receive d phi(q) and
// d keff in fp32 when out_f32 (chain rule by the caller).
static void vec_backward(const lmoe_lsm_desc& dd, const BwdPlan& w, int B, int N, int H, int D, const void* phq,
                         const void* phk, const void* v, const void* a_pre, const void* dO, const float* M0,
                         const float* dM_final, void* dq, void* dk, void* dv, void* da, float* dM0, bool out_f32,
                         uint8_t* ws, cudaStream_t st) {
    using bf = __nv_bfloat16;
    const int nchunk = (N + lmoe_dev::kC - 1) / lmoe_dev::kC;
    const bool hg = dd.instance == LMOE_HGRN2;
    LsmCall c{&dd, B, N, N, H, D, LMOE_BF16, phq, phk, v, nullptr, nullptr, nullptr, ws, w.pl, st, a_pre};
    c.setup();
    c.clear_err();
    lmoe_dev::VecBwdParams vp{};
    vp.B = B; vp.N = N; vp.H = H;
    vp.seg_len = w.pl.seg_len; vp.nseg = w.pl.nseg; vp.nchunk = nchunk;
    vp.Min = c.p.Min;
    vp.bd = reinterpret_cast<const float*>(ws + w.off_bd);
    vp.dq = dq; vp.dk = dk;
    vp.dv = static_cast<bf*>(dv);
    vp.da = static_cast<bf*>(da);
    vp.out_f32 = out_f32 ? 1 : 0;
    vp.err = c.p.err;
    vp.trace = c.p.trace;
    bf* snapM = reinterpret_cast<bf*>(ws + w.off_mst);
    bf* snapX = reinterpret_cast<bf*>(ws + w.off_dmst);
    const CUtensorMap tq = c.tmap<bf>(phq), tk = c.tmap<bf>(phk), tv = c.tmap<bf>(v), tdo = c.tmap<bf>(dO),
                      ta = c.tmap<bf>(a_pre);
    const dim3 sgrid(w.pl.nseg, H, B);
    // 1-2: states entering every chunk (forward)
    c.state_pass<bf>();
    c.combine(M0, nullptr, true, nullptr, nullptr, nullptr, 0);
    vp.snap = snapM;
    LMOE_CUDA_CHECK(lmoe_dev::launch_vec_carry(hg, false, sgrid, st, tk, tv, ta, vp));
    // 3-4: adjoints leaving every chunk (reverse), dM0
    LsmCall r = c;
    r.k = phq;
    r.v = dO;
    r.var.rev = 1;
    r.state_pass<bf>();
    r.combine(dM_final, nullptr, true, dM0, nullptr, nullptr, 0, 1);
    vp.snap = snapX;
    vp.snap_fwd = snapM;  // 5: the REV carry also forms the gate gradient's boundary terms
    vp.bd_out = reinterpret_cast<float*>(ws + w.off_bd);
    LMOE_CUDA_CHECK(lmoe_dev::launch_vec_carry(false, true, sgrid, st, tq, tdo, ta, vp));
    const long long rows = (long long)B * H * (nchunk + 1) * D;
    // 6: fused chunk backward
    // bf16 outputs leave through TMA bulk stores (dq / dk only when not fp32 intermediates)
    const CUtensorMap tm[11] = {tq, tk, tv, tdo, ta,
                                make_tmap_2d(snapM, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, rows, D, 64, 128),
                                make_tmap_2d(snapX, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, rows, D, 64, 128),
                                out_f32 ? tq : c.tmap<bf>(dq), out_f32 ? tk : c.tmap<bf>(dk), c.tmap<bf>(dv),
                                c.tmap<bf>(da)};
    if (hg && !out_f32)  // HGRN2's effective key 1 - sigmoid(a) ignores k
        LMOE_CUDA_CHECK(cudaMemsetAsync(dk, 0, (size_t)B * N * H * D * sizeof(bf), st));
    vp.pf_ahead = env_int("LMOE_VB_PF", 0) * num_sms();  // developer A/B knob (measured: no gain, off)
    LMOE_CUDA_CHECK(lmoe_dev::launch_vec_bwd_chunk(hg, dim3(nchunk, H, B), st, tm, vp));
    g_launch_count += 3;
    c.check_err();
}
}  // namespace lmoe_host

namespace lmoe_host {
// Normaliser backward (lsm.hpp:584-596): o = num / den.  The tape's VJP is the sum of the
// backward of the unnormalised LSM under dnum = dO / den and the backward of the LSM with
// value e0 (whose output column 0 is den) under dden = -(dO . num) / den^2: two forwards
// (num, den), one elementwise split, two backward calls, one accumulation.
struct NormPlan {
    size_t off_inner = 0, inner = 0, off_fwd = 0, fwd = 0, off_e0 = 0, off_num = 0, off_den = 0, off_dO1 = 0,
           off_dO2 = 0, off_dq2 = 0, off_dk2 = 0, off_dv2 = 0, off_da2 = 0, off_err = 0, total = 0;
};
static NormPlan plan_norm(const lmoe_lsm_desc* d, int B, int N, int H, int D, lmoe_dtype dt) {
    lmoe_lsm_desc dd = *d;
    dd.use_normalizer = 0;
    NormPlan p;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    p.inner = plan_bwd(&dd, B, N, H, D, dt).total;
    p.off_inner = take(p.inner);
    p.fwd = plan_lsm(B, N, H, D).total;
    p.off_fwd = take(p.fwd);
    const size_t act = (size_t)B * N * H * D * (dt == LMOE_BF16 ? 2 : 4);
    p.off_e0 = take(act); p.off_num = take(act); p.off_den = take(act);
    p.off_dO1 = take(act); p.off_dO2 = take(act);
    p.off_dq2 = take(act); p.off_dk2 = take(act); p.off_dv2 = take(act); p.off_da2 = take(act);
    p.off_err = take(64);
    p.total = off;
    return p;
}
}  // namespace lmoe_host

extern "C" size_t lmoe_lsm_bwd_workspace_size(const lmoe_lsm_desc* desc, int B, int N, int H, int D,
                                              lmoe_dtype dtype) {
    if (!desc || B < 1 || N < 1 || H < 1 || D < 1) return 0;
    if (desc->use_normalizer) return plan_norm(desc, B, N, H, D, dtype).total;
    return plan_bwd(desc, B, N, H, D, dtype).total;
}

extern "C" int lmoe_lsm_bwd(const lmoe_lsm_desc* desc, int B, int N, int H, int D, lmoe_dtype dtype,
                            const void* q, const void* k, const void* v, const void* a_pre,
                            const float* b_pre, const float* a_raw, const float* M0, const void* dO,
                            const float* dM_final, void* dq, void* dk, void* dv, void* da_pre,
                            float* db_pre, float* da_raw, float* dM0, void* workspace,
                            size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        validate(desc, B, N, H, D, dtype, q, k, v, dO);
        if (!dq || !dk || !dv) throw Error(LMOE_ERR_ARG, "lmoe_lsm_bwd: null gradient tensor");
        const int mode = device_decay_mode(desc->instance);
        if (desc->use_normalizer) {
            if (mode == lmoe_dev::kDecayTokenVector && (!a_pre || !da_pre))
                throw Error(LMOE_ERR_ARG, "lmoe_lsm_bwd: TokenVector instances need a_pre and da_pre");
            const NormPlan w = plan_norm(desc, B, N, H, D, dtype);
            if (!workspace || workspace_bytes < w.total)
                throw Error(LMOE_ERR_ARG, "lmoe_lsm_bwd: workspace too small (need " + std::to_string(w.total) + " bytes)");
            uint8_t* ws = static_cast<uint8_t*>(workspace);
            cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
            const bool bf16 = dtype == LMOE_BF16;
            const size_t rows = (size_t)B * N * H;
            lmoe_lsm_desc dd = *desc;
            dd.use_normalizer = 0;
            auto chk = [](int rc) {
                if (rc != LMOE_OK) throw Error(rc, lmoe_last_error());
            };
            int* err = reinterpret_cast<int*>(ws + w.off_err);
            LMOE_CUDA_CHECK(cudaMemsetAsync(err, 0, 64, st));
            void* e0 = ws + w.off_e0;
            LMOE_CUDA_CHECK(lmoe_dev::launch_norm_helpers(0, bf16, e0, nullptr, nullptr, nullptr, nullptr, nullptr,
                                                          rows, D, nullptr, st));
            chk(lmoe_lsm_fwd(&dd, B, N, H, D, dtype, q, k, v, a_pre, b_pre, a_raw, M0, nullptr, ws + w.off_num,
                             nullptr, nullptr, ws + w.off_fwd, w.fwd, stream));
            chk(lmoe_lsm_fwd(&dd, B, N, H, D, dtype, q, k, e0, a_pre, b_pre, a_raw, nullptr, nullptr,
                             ws + w.off_den, nullptr, nullptr, ws + w.off_fwd, w.fwd, stream));
            LMOE_CUDA_CHECK(lmoe_dev::launch_norm_helpers(1, bf16, nullptr, ws + w.off_num, ws + w.off_den, dO,
                                                          ws + w.off_dO1, ws + w.off_dO2, rows, D, err, st));
            g_launch_count += 2;
            if (desc->flags & LMOE_FLAG_CHECK) {
                int e = 0;
                LMOE_CUDA_CHECK(cudaMemcpyAsync(&e, err, sizeof(int), cudaMemcpyDeviceToHost, st));
                LMOE_CUDA_CHECK(cudaStreamSynchronize(st));
                if (e)
                    throw Error(LMOE_ERR_DEGENERATE,
                                std::string("degenerate normalizer in instance ") + instance_name(desc->instance));
            }
            const bool vec = mode == lmoe_dev::kDecayTokenVector;
            chk(lmoe_lsm_bwd(&dd, B, N, H, D, dtype, q, k, v, a_pre, b_pre, a_raw, M0, ws + w.off_dO1, dM_final,
                             dq, dk, dv, da_pre, db_pre, da_raw, dM0, ws + w.off_inner, w.inner, stream));
            chk(lmoe_lsm_bwd(&dd, B, N, H, D, dtype, q, k, e0, a_pre, b_pre, a_raw, nullptr, ws + w.off_dO2, nullptr,
                             ws + w.off_dq2, ws + w.off_dk2, ws + w.off_dv2, vec ? ws + w.off_da2 : nullptr, nullptr,
                             nullptr, nullptr, ws + w.off_inner, w.inner, stream));
            LMOE_CUDA_CHECK(lmoe_dev::launch_norm_helpers(2, bf16, dq, ws + w.off_dq2, nullptr, nullptr, nullptr,
                                                          nullptr, rows, D, nullptr, st));
            LMOE_CUDA_CHECK(lmoe_dev::launch_norm_helpers(2, bf16, dk, ws + w.off_dk2, nullptr, nullptr, nullptr,
                                                          nullptr, rows, D, nullptr, st));
            g_launch_count += 3;
            if (vec) {
                LMOE_CUDA_CHECK(lmoe_dev::launch_norm_helpers(2, bf16, da_pre, ws + w.off_da2, nullptr, nullptr, nullptr,
                                                              nullptr, rows, D, nullptr, st));
                ++g_launch_count;
            }
            return;
        }
        if (mode == lmoe_dev::kDecayTokenVector) {
            if (dtype != LMOE_BF16)
                throw Error(LMOE_ERR_UNSUPPORTED, std::string("lmoe_lsm_bwd: instance ") + instance_name(desc->instance) +
                                                      " has a device backward for bf16 / head_dim 128 only");
            if (!a_pre || !da_pre) throw Error(LMOE_ERR_ARG, "lmoe_lsm_bwd: TokenVector instances need a_pre and da_pre");
        }
        const bool mamba = mode == lmoe_dev::kDecayTokenScalar;
        if (mamba && (!db_pre || !da_raw)) throw Error(LMOE_ERR_ARG, "lmoe_lsm_bwd: Mamba2 needs db_pre and da_raw");
        const BwdPlan w = plan_bwd(desc, B, N, H, D, dtype);
        if (!workspace || workspace_bytes < w.total)
            throw Error(LMOE_ERR_ARG, "lmoe_lsm_bwd: workspace too small (need " + std::to_string(w.total) + " bytes)");
        uint8_t* ws = static_cast<uint8_t*>(workspace);
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const bool bf16 = dtype == LMOE_BF16;
        const size_t act = (size_t)B * N * H * D;
        const int BH = B * H;
        auto F = [&](size_t off) { return reinterpret_cast<float*>(ws + off); };
        // the chunk passes run with identity feature map and no normaliser
        lmoe_lsm_desc dd = *desc;
        dd.feature_map = 0;
        dd.use_normalizer = 0;
        const void* phq = q;
        const void* phk = k;
        if (desc->feature_map != 0) {
            LMOE_CUDA_CHECK(lmoe_dev::launch_apply_fmap(bf16, desc->feature_map, q, ws + w.off_phq, act, st));
            LMOE_CUDA_CHECK(lmoe_dev::launch_apply_fmap(bf16, desc->feature_map, k, ws + w.off_phk, act, st));
            g_launch_count += 2;
            phq = ws + w.off_phq;
            phk = ws + w.off_phk;
        }
        const int nchunk = (N + lmoe_dev::kC - 1) / lmoe_dev::kC;
        float* dphq = F(w.off_dphq);
        float* dkef = F(w.off_dkef);
        const bool direct = desc->feature_map == 0;
        if (mode == lmoe_dev::kDecayTokenVector) {
            vec_backward(dd, w, B, N, H, D, phq, phk, v, a_pre, dO, M0, dM_final, direct ? dq : dphq,
                         direct ? dk : dkef, dv, da_pre, dM0, !direct, ws, st);
            if (!direct) {
                LMOE_CUDA_CHECK(lmoe_dev::launch_bwd_finish(bf16, desc->feature_map, false, q, k, dphq, dkef, nullptr,
                                                            dq, dk, F(w.off_dkf), B, N, H, st));
                ++g_launch_count;
            }
            if (desc->flags & LMOE_FLAG_CHECK) LMOE_CUDA_CHECK(cudaStreamSynchronize(st));
            return;
        }
        const float* M0T = nullptr;
        if (M0) {
            LMOE_CUDA_CHECK(lmoe_dev::launch_transpose_states(M0, F(w.off_M0T), BH, D, st));
            ++g_launch_count;
            M0T = F(w.off_M0T);
        }
        const float* dMfT = nullptr;
        if (dM_final) {
            LMOE_CUDA_CHECK(lmoe_dev::launch_transpose_states(dM_final, F(w.off_dMfT), BH, D, st));
            ++g_launch_count;
            dMfT = F(w.off_dMfT);
        }
        // side: 1 / 2 = write the per-chunk state operands (dq pass: M_c^T, dk pass: dM_c^T)
        // shared_T (the dv pass): its keys / values are the dk pass's values / keys with the same
        // reverse-time decay weights, so its segment states, carried-in states and final state
        // are the transposes of the dk pass's (no state pass, no combine; the initial states
        // dM_final and dM_final^T are transposes too)
        auto pass = [&](const void* qq, const void* kk, const void* vv, void* oo, bool rev, bool out_f32,
                        bool kfq, const float* init, float* fin, int side, bool shared_T = false) {
            LsmCall c{&dd, B, N, N, H, D, dtype, qq, kk, vv, b_pre, a_raw, oo, ws, w.pl, st, nullptr};
            c.setup();
            c.var.rev = rev ? 1 : 0;
            c.p.out_f32 = out_f32 ? 1 : 0;
            c.p.rev_kfq = kfq ? 1 : 0;
            c.p.nchunk_tot = nchunk;
            if (mamba && side == 1) c.p.mst = ws + w.off_mst;
            if (mamba && side == 2) c.p.mst = ws + w.off_dmst;
            c.clear_err();
            if (shared_T) {
                float* minT = c.p.Sseg;  // the segment-state region is free in this pass
                c.mark();  // phase-timer layout of a pass: the "state pass" is the transposes
                LMOE_CUDA_CHECK(lmoe_dev::launch_transpose_states(c.p.Min, minT, BH * w.pl.nseg, D, st));
                if (fin) LMOE_CUDA_CHECK(lmoe_dev::launch_transpose_states(F(w.off_dkfin), fin, BH, D, st));
                g_launch_count += fin ? 2 : 1;
                c.p.Min = minT;
                c.mark();
            } else {
                if (bf16) c.state_pass<__nv_bfloat16>(); else c.state_pass<float>();
                c.combine(init, nullptr, true, fin, nullptr, nullptr, 0, rev ? 1 : 0);
            }
            if (bf16) c.output_pass<__nv_bfloat16>(); else c.output_pass<float>();
            c.finish_timing();
            c.check_err();
        };
        // identity feature map: dq = dphi(q) and dk = kf dkeff come straight out of the dq / dk
        // passes (the kf row scale of the REV epilogue), in the input dtype; otherwise fp32
        // intermediates go through the chain-rule kernel
        pass(dO, v, phk, direct ? dq : dphq, false, !direct, false, M0T, F(w.off_MfinT), 1);
        pass(v, dO, phq, direct ? dk : dkef, true, !direct, direct && mamba, dMfT, dM0 ? F(w.off_dkfin) : nullptr, 2);
        pass(phk, phq, dO, dv, true, false, mamba, dM_final, dM0, 0, true);
        if (!direct) {
            LMOE_CUDA_CHECK(lmoe_dev::launch_bwd_finish(bf16, desc->feature_map, mamba, q, k, dphq, dkef, b_pre, dq,
                                                        dk, F(w.off_dkf), B, N, H, st));
            ++g_launch_count;
        }
        if (mamba) {
            LsmCall c{&dd, B, N, N, H, D, dtype, q, k, v, b_pre, a_raw, nullptr, ws, w.pl, st, nullptr};
            const CUtensorMapDataType tdt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
            const int esz = bf16 ? 2 : 4, epb = 128 / esz;
            const uint64_t srows = (uint64_t)BH * nchunk * D;
            const CUtensorMap tm = make_tmap_2d(ws + w.off_mst, tdt, esz, D, srows, D, epb, D);
            const CUtensorMap tdm = make_tmap_2d(ws + w.off_dmst, tdt, esz, D, srows, D, epb, D);
            CUtensorMap tq, tk, tv, tdo;
            if (bf16) {
                tq = c.tmap<__nv_bfloat16>(phq); tk = c.tmap<__nv_bfloat16>(phk);
                tv = c.tmap<__nv_bfloat16>(v); tdo = c.tmap<__nv_bfloat16>(dO);
            } else {
                tq = c.tmap<float>(phq); tk = c.tmap<float>(phk); tv = c.tmap<float>(v); tdo = c.tmap<float>(dO);
            }
            LMOE_CUDA_CHECK(lmoe_dev::launch_mamba_dgate(bf16, tq, tk, tv, tdo, tm, tdm, b_pre, a_raw,
                                                         direct ? nullptr : F(w.off_dkf), direct ? dk : nullptr,
                                                         db_pre, da_raw, B, N, H, st));
            ++g_launch_count;
        }
        if (desc->flags & LMOE_FLAG_CHECK) LMOE_CUDA_CHECK(cudaStreamSynchronize(st));
    });
}

// Developer aid: copies the clock64 phase trace of the last LMOE_TRACE run (64 x 16 u64).
extern "C" int lmoe_debug_trace_read(unsigned long long* out) {
    return guarded([&]() {
        if (!g_trace) throw Error(LMOE_ERR_ARG, "no trace (set LMOE_TRACE)");
        LMOE_CUDA_CHECK(cudaDeviceSynchronize());
        LMOE_CUDA_CHECK(cudaMemcpy(out, g_trace, (64 * 16 + 4 * 4096) * 8, cudaMemcpyDeviceToHost));
    });
}

// ------------------------------------------------------------------- SP backward (8(f) rank 1)
namespace lmoe_host {
struct SpBwdPlan {
    SpWorkspace f;  // forward payload, gather, M0
    size_t off_bpay = 0, off_bgath = 0, off_Xin = 0, off_phq = 0, off_dar = 0, off_bws = 0, bws = 0, total = 0;
};
static size_t bwd_payload_floats(const lmoe_lsm_desc* d, int D) { return (size_t)D * D + payload_lw(d, D); }

static SpBwdPlan plan_sp_bwd(const lmoe_lsm_desc* d, int B, int N_local, int H, int D, lmoe_dtype dt, int world,
                            int n_min = -1) {
    SpBwdPlan p;
    p.f = plan_sp(d, B, N_local, H, D, world, n_min);
    size_t off = align_up(p.f.total, 256);
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    const size_t BH = (size_t)B * H, P = BH * bwd_payload_floats(d, D);
    p.off_bpay = take(P * 4);
    p.off_bgath = take((size_t)world * P * 4);
    p.off_Xin = take(BH * D * D * 4);
    if (d->feature_map != 0) p.off_phq = take((size_t)B * N_local * H * D * (dt == LMOE_BF16 ? 2 : 4));
    p.off_dar = take((size_t)H * 4);
    p.bws = plan_bwd(d, B, N_local, H, D, dt).total;
    if (n_min > 0 && n_min != N_local) p.bws = std::max(p.bws, plan_bwd(d, B, n_min, H, D, dt).total);
    p.off_bws = take(p.bws);
    p.total = off;
    return p;
}

// Normaliser SP backward (sp_norm_bwd below): o = num / den with num = LSM(q, k, v) and den =
// column 0 of LSM(q, k, e0), both unnormalised and sequence-parallel (den's state column 0 is
// the normaliser z, lsm.hpp:584-596), so the VJP is the unnormalised SP backward of num under
// dO / den plus that of den under -(dO . num) / den^2 -- the composition lmoe_lsm_bwd uses
// locally, with the SP forward / backward (and their collectives) in place of the local ones.
struct SpNormPlan {
    size_t off_e0 = 0, off_num = 0, off_den = 0, off_dO1 = 0, off_dO2 = 0, off_dq2 = 0, off_dk2 = 0, off_dv2 = 0,
           off_da2 = 0, off_err = 0, off_inner = 0, inner = 0, total = 0;
};
static SpNormPlan plan_sp_norm(size_t rows, int D, lmoe_dtype dt, size_t inner) {
    SpNormPlan p;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    p.inner = inner;
    p.off_inner = take(inner);
    const size_t act = rows * D * (dt == LMOE_BF16 ? 2 : 4);
    p.off_e0 = take(act); p.off_num = take(act); p.off_den = take(act);
    p.off_dO1 = take(act); p.off_dO2 = take(act);
    p.off_dq2 = take(act); p.off_dk2 = take(act); p.off_dv2 = take(act); p.off_da2 = take(act);
    p.off_err = take(64);
    p.total = off;
    return p;
}
// fwd(desc, v, out, ws, bytes) and bwd(desc, v, dO, dq, dk, dv, da, dM0, ws, bytes) run the
// unnormalised SP forward / backward of this rank (or of all virtual ranks)
template <typename Fwd, typename Bwd>
static void sp_norm_bwd(const lmoe_lsm_desc* desc, size_t rows, int D, lmoe_dtype dt, const void* v, const void* dO,
                        void* dq, void* dk, void* dv, void* da_pre, float* dM0, uint8_t* ws, const SpNormPlan& w,
                        cudaStream_t st, Fwd fwd, Bwd bwd) {
    lmoe_lsm_desc dd = *desc;
    dd.use_normalizer = 0;
    const bool bf16 = dt == LMOE_BF16;
    const bool vec = device_decay_mode(desc->instance) == lmoe_dev::kDecayTokenVector;
    int* err = reinterpret_cast<int*>(ws + w.off_err);
    LMOE_CUDA_CHECK(cudaMemsetAsync(err, 0, 64, st));
    void* e0 = ws + w.off_e0;
    LMOE_CUDA_CHECK(lmoe_dev::launch_norm_helpers(0, bf16, e0, nullptr, nullptr, nullptr, nullptr, nullptr, rows, D,
                                                  nullptr, st));
    fwd(&dd, v, ws + w.off_num);
    fwd(&dd, e0, ws + w.off_den);
    LMOE_CUDA_CHECK(lmoe_dev::launch_norm_helpers(1, bf16, nullptr, ws + w.off_num, ws + w.off_den, dO, ws + w.off_dO1,
                                                  ws + w.off_dO2, rows, D, err, st));
    g_launch_count += 2;
    if (desc->flags & LMOE_FLAG_CHECK) {
        int e = 0;
        LMOE_CUDA_CHECK(cudaMemcpyAsync(&e, err, sizeof(int), cudaMemcpyDeviceToHost, st));
        LMOE_CUDA_CHECK(cudaStreamSynchronize(st));
        if (e)
            throw Error(LMOE_ERR_DEGENERATE, std::string("degenerate normalizer in instance ") + instance_name(desc->instance));
    }
    bwd(&dd, v, ws + w.off_dO1, dq, dk, dv, da_pre, dM0);
    bwd(&dd, e0, ws + w.off_dO2, ws + w.off_dq2, ws + w.off_dk2, ws + w.off_dv2, vec ? ws + w.off_da2 : nullptr,
        nullptr);
    LMOE_CUDA_CHECK(lmoe_dev::launch_norm_helpers(2, bf16, dq, ws + w.off_dq2, nullptr, nullptr, nullptr, nullptr, rows,
                                                  D, nullptr, st));
    LMOE_CUDA_CHECK(lmoe_dev::launch_norm_helpers(2, bf16, dk, ws + w.off_dk2, nullptr, nullptr, nullptr, nullptr, rows,
                                                  D, nullptr, st));
    g_launch_count += 2;
    if (vec) {
        LMOE_CUDA_CHECK(lmoe_dev::launch_norm_helpers(2, bf16, da_pre, ws + w.off_da2, nullptr, nullptr, nullptr,
                                                      nullptr, rows, D, nullptr, st));
        ++g_launch_count;
    }
}
static void check_sp_bwd_args(const lmoe_lsm_desc* d) { (void)d; }

// One slice: writes the forward payload [M | log D] (from zero) and the reverse-time payload
// [X | log D] (X = sum_t (phi(q_t) e^{P_t})^T dO_t, P_t = decay from the slice start through t).
template <typename T>
static void sp_bwd_payloads(const lmoe_lsm_desc* d, int B, int n, int Nstride, int H, int D, lmoe_dtype dt,
                            const void* q, const void* k, const void* v, const void* a_pre, const float* b_pre,
                            const float* a_raw, const void* dO, uint8_t* ws, const SpBwdPlan& w, float* fpay,
                            float* bpay, cudaStream_t st) {
    LsmCall c{d, B, n, Nstride, H, D, dt, q, k, v, b_pre, a_raw, nullptr, ws, plan_lsm(B, n, H, D), st, a_pre};
    c.setup();
    sp_phase_a<T>(c, fpay);
    // reverse pass over (phi(q), dO): identity map (phi applied beforehand), no normaliser
    lmoe_lsm_desc dd = *d;
    dd.feature_map = 0;
    dd.use_normalizer = 0;
    const void* phq = q;
    if (d->feature_map != 0) {
        LMOE_CUDA_CHECK(lmoe_dev::launch_apply_fmap(dt == LMOE_BF16, d->feature_map, q, ws + w.off_phq,
                                                    (size_t)B * n * H * D, st));  // B == 1 or dense
        ++g_launch_count;
        phq = ws + w.off_phq;
    }
    LsmCall r{&dd, B, n, Nstride, H, D, dt, q, phq, dO, b_pre, a_raw, nullptr, ws, plan_lsm(B, n, H, D), st, a_pre};
    r.setup();
    r.var.rev = 1;
    const int P = (int)bwd_payload_floats(d, D);
    r.state_pass<T>();
    r.combine(nullptr, nullptr, false, bpay, nullptr, bpay + P - r.lw, P, 1);
}
}  // namespace lmoe_host

static SpNormPlan plan_sp_norm_rank(const lmoe_lsm_desc* desc, int B, int N_local, int H, int D, lmoe_dtype dtype,
                                    int world) {
    lmoe_lsm_desc dd = *desc;
    dd.use_normalizer = 0;
    const size_t inner = std::max(plan_sp_bwd(&dd, B, N_local, H, D, dtype, world).total,
                                  plan_sp(&dd, B, N_local, H, D, world).total);
    return plan_sp_norm((size_t)B * N_local * H, D, dtype, inner);
}

extern "C" size_t lmoe_sp_lsm_bwd_workspace_size(const lmoe_lsm_desc* desc, int B, int N_local, int H, int D,
                                                 lmoe_dtype dtype, int world) {
    if (!desc || B < 1 || N_local < 1 || H < 1 || D < 1 || world < 1) return 0;
    if (desc->use_normalizer) return plan_sp_norm_rank(desc, B, N_local, H, D, dtype, world).total;
    return plan_sp_bwd(desc, B, N_local, H, D, dtype, world).total;
}

extern "C" int lmoe_sp_lsm_bwd(const lmoe_lsm_desc* desc, int B, int N_local, int H, int D, lmoe_dtype dtype,
                               const void* q, const void* k, const void* v, const void* a_pre, const float* b_pre,
                               const float* a_raw, const void* dO, void* dq, void* dk, void* dv, void* da_pre,
                               float* db_pre, float* da_raw, float* dM0, void* nccl_comm, int rank, int world,
                               void* workspace, size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        validate(desc, B, N_local, H, D, dtype, q, k, v, dO);
        check_sp_bwd_args(desc);
        if (world < 1 || rank < 0 || rank >= world) throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_bwd: bad rank");
        if (world > 1 && !nccl_comm) throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_bwd: null communicator");
        if (desc->use_normalizer) {
            const SpNormPlan w = plan_sp_norm_rank(desc, B, N_local, H, D, dtype, world);
            if (!workspace || workspace_bytes < w.total)
                throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_bwd: workspace too small (need " + std::to_string(w.total) + " bytes)");
            uint8_t* ws = static_cast<uint8_t*>(workspace);
            auto chk = [](int rc) {
                if (rc != LMOE_OK) throw Error(rc, lmoe_last_error());
            };
            auto fwd = [&](const lmoe_lsm_desc* dd, const void* vv, void* out) {
                chk(lmoe_sp_lsm_fwd(dd, B, N_local, H, D, dtype, q, k, vv, a_pre, b_pre, a_raw, out, nullptr, nullptr,
                                    nccl_comm, rank, world, ws + w.off_inner, w.inner, stream));
            };
            auto bwd = [&](const lmoe_lsm_desc* dd, const void* vv, const void* g, void* gq, void* gk, void* gv,
                           void* ga, float* gM0) {
                chk(lmoe_sp_lsm_bwd(dd, B, N_local, H, D, dtype, q, k, vv, a_pre, b_pre, a_raw, g, gq, gk, gv, ga,
                                    db_pre, da_raw, gM0, nccl_comm, rank, world, ws + w.off_inner, w.inner, stream));
            };
            sp_norm_bwd(desc, (size_t)B * N_local * H, D, dtype, v, dO, dq, dk, dv, da_pre, dM0, ws, w,
                        reinterpret_cast<cudaStream_t>(stream), fwd, bwd);
            return;
        }
        const SpBwdPlan w = plan_sp_bwd(desc, B, N_local, H, D, dtype, world);
        if (!workspace || workspace_bytes < w.total)
            throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_bwd: workspace too small (need " + std::to_string(w.total) + " bytes)");
        uint8_t* ws = static_cast<uint8_t*>(workspace);
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const int BH = B * H;
        const size_t Pf = (size_t)BH * payload_floats(desc, D), Pb = (size_t)BH * bwd_payload_floats(desc, D);
        float* fpay = reinterpret_cast<float*>(ws + w.f.off_payload);
        float* fgath = reinterpret_cast<float*>(ws + w.f.off_gathered);
        float* bpay = reinterpret_cast<float*>(ws + w.off_bpay);
        float* bgath = reinterpret_cast<float*>(ws + w.off_bgath);
        float* M0 = reinterpret_cast<float*>(ws + w.f.off_M0);
        float* Xin = reinterpret_cast<float*>(ws + w.off_Xin);
        if (dtype == LMOE_BF16)
            sp_bwd_payloads<__nv_bfloat16>(desc, B, N_local, N_local, H, D, dtype, q, k, v, a_pre, b_pre, a_raw, dO,
                                           ws, w, fpay, bpay, st);
        else
            sp_bwd_payloads<float>(desc, B, N_local, N_local, H, D, dtype, q, k, v, a_pre, b_pre, a_raw, dO, ws, w,
                                   fpay, bpay, st);
        if (nccl_comm) {
            NCCL_CHECK(ncclGroupStart());
            NCCL_CHECK(ncclAllGather(fpay, fgath, Pf, ncclFloat, static_cast<ncclComm_t>(nccl_comm), st));
            NCCL_CHECK(ncclAllGather(bpay, bgath, Pb, ncclFloat, static_cast<ncclComm_t>(nccl_comm), st));
            NCCL_CHECK(ncclGroupEnd());
        } else {
            LMOE_CUDA_CHECK(cudaMemcpyAsync(fgath, fpay, Pf * 4, cudaMemcpyDeviceToDevice, st));
            LMOE_CUDA_CHECK(cudaMemcpyAsync(bgath, bpay, Pb * 4, cudaMemcpyDeviceToDevice, st));
        }
        g_last_gather_elements = (long long)world * (long long)(Pf + Pb);
        const int lw = payload_lw(desc, D);
        LMOE_CUDA_CHECK(lmoe_dev::launch_rank_combine(dim3((D * D + 255) / 256, BH), st, fgath,
                                                      (int)payload_floats(desc, D), BH, rank, D, D, 0, lw, M0,
                                                      nullptr));
        LMOE_CUDA_CHECK(lmoe_dev::launch_rank_combine_rev(bgath, (int)bwd_payload_floats(desc, D), BH, rank, world,
                                                          D, D, lw, Xin, st));
        g_launch_count += 2;
        const int rc = lmoe_lsm_bwd(desc, B, N_local, H, D, dtype, q, k, v, a_pre, b_pre, a_raw, M0, dO, Xin, dq,
                                    dk, dv, da_pre, db_pre, da_raw, dM0, ws + w.off_bws, w.bws, stream);
        if (rc != LMOE_OK) throw Error(rc, lmoe_last_error());
    });
}

static SpNormPlan plan_sp_norm_loopback(const lmoe_lsm_desc* desc, int B, int N, int H, int D, lmoe_dtype dtype,
                                        int world) {
    lmoe_lsm_desc dd = *desc;
    dd.use_normalizer = 0;
    const int n = (N + world - 1) / world;
    const size_t inner = std::max(plan_sp_bwd(&dd, B, n, H, D, dtype, world, N / world).total,
                                  plan_sp(&dd, B, n, H, D, world, N / world).total);
    return plan_sp_norm((size_t)B * N * H, D, dtype, inner);
}

extern "C" size_t lmoe_sp_lsm_bwd_loopback_workspace_size(const lmoe_lsm_desc* desc, int B, int N, int H, int D,
                                                          lmoe_dtype dtype, int world) {
    if (!desc || world < 1 || N < world) return 0;
    if (desc->use_normalizer) return plan_sp_norm_loopback(desc, B, N, H, D, dtype, world).total;
    return plan_sp_bwd(desc, B, (N + world - 1) / world, H, D, dtype, world, N / world).total;
}

extern "C" int lmoe_sp_lsm_bwd_loopback(const lmoe_lsm_desc* desc, int B, int N, int H, int D, lmoe_dtype dtype,
                                        const void* q, const void* k, const void* v, const void* a_pre,
                                        const float* b_pre, const float* a_raw, const void* dO, void* dq, void* dk,
                                        void* dv, void* da_pre, float* db_pre, float* da_raw, float* dM0, int world,
                                        void* workspace, size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        validate(desc, B, N, H, D, dtype, q, k, v, dO);
        check_sp_bwd_args(desc);
        if (B != 1) throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_bwd_loopback: B == 1 (rank slices are contiguous rows)");
        if (world < 1 || N < world) throw Error(LMOE_ERR_ARG, "chunk_range: need at least one row per rank");
        if (desc->use_normalizer) {
            const SpNormPlan w = plan_sp_norm_loopback(desc, B, N, H, D, dtype, world);
            if (!workspace || workspace_bytes < w.total)
                throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_bwd_loopback: workspace too small");
            uint8_t* ws = static_cast<uint8_t*>(workspace);
            auto chk = [](int rc) {
                if (rc != LMOE_OK) throw Error(rc, lmoe_last_error());
            };
            auto fwd = [&](const lmoe_lsm_desc* dd, const void* vv, void* out) {
                chk(lmoe_sp_lsm_fwd_loopback(dd, B, N, H, D, dtype, q, k, vv, a_pre, b_pre, a_raw, out, nullptr,
                                             nullptr, world, ws + w.off_inner, w.inner, stream));
            };
            auto bwd = [&](const lmoe_lsm_desc* dd, const void* vv, const void* g, void* gq, void* gk, void* gv,
                           void* ga, float* gM0) {
                chk(lmoe_sp_lsm_bwd_loopback(dd, B, N, H, D, dtype, q, k, vv, a_pre, b_pre, a_raw, g, gq, gk, gv, ga,
                                             db_pre, da_raw, gM0, world, ws + w.off_inner, w.inner, stream));
            };
            sp_norm_bwd(desc, (size_t)B * N * H, D, dtype, v, dO, dq, dk, dv, da_pre, dM0, ws, w,
                        reinterpret_cast<cudaStream_t>(stream), fwd, bwd);
            return;
        }
        const SpBwdPlan w = plan_sp_bwd(desc, B, (N + world - 1) / world, H, D, dtype, world, N / world);
        if (!workspace || workspace_bytes < w.total)
            throw Error(LMOE_ERR_ARG, "lmoe_sp_lsm_bwd_loopback: workspace too small");
        uint8_t* ws = static_cast<uint8_t*>(workspace);
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const bool bf16 = dtype == LMOE_BF16;
        const size_t esz = bf16 ? 2 : 4;
        const int BH = B * H;
        const size_t Pf = (size_t)BH * payload_floats(desc, D), Pb = (size_t)BH * bwd_payload_floats(desc, D);
        float* fgath = reinterpret_cast<float*>(ws + w.f.off_gathered);
        float* bgath = reinterpret_cast<float*>(ws + w.off_bgath);
        float* M0 = reinterpret_cast<float*>(ws + w.f.off_M0);
        float* Xin = reinterpret_cast<float*>(ws + w.off_Xin);
        float* dar = reinterpret_cast<float*>(ws + w.off_dar);
        auto slice = [&](int r, int& r0, int& len) {  // chunk_range (parallel.hpp:192-197)
            const int base = N / world, rem = N % world;
            r0 = r * base + std::min(r, rem);
            len = base + (r < rem ? 1 : 0);
        };
        auto at = [&](const void* p, int r0, size_t e) -> const void* {
            return p ? static_cast<const uint8_t*>(p) + (size_t)r0 * H * D * e : nullptr;
        };
        auto atw = [&](void* p, int r0, size_t e) -> void* {
            return p ? static_cast<uint8_t*>(p) + (size_t)r0 * H * D * e : nullptr;
        };
        for (int r = 0; r < world; ++r) {
            int r0, len;
            slice(r, r0, len);
            const float* bp = b_pre ? b_pre + (size_t)r0 * H : nullptr;
            if (bf16)
                sp_bwd_payloads<__nv_bfloat16>(desc, B, len, len, H, D, dtype, at(q, r0, esz), at(k, r0, esz),
                                               at(v, r0, esz), at(a_pre, r0, esz), bp, a_raw, at(dO, r0, esz), ws, w,
                                               fgath + r * Pf, bgath + r * Pb, st);
            else
                sp_bwd_payloads<float>(desc, B, len, len, H, D, dtype, at(q, r0, esz), at(k, r0, esz),
                                       at(v, r0, esz), at(a_pre, r0, esz), bp, a_raw, at(dO, r0, esz), ws, w,
                                       fgath + r * Pf, bgath + r * Pb, st);
        }
        g_last_gather_elements = (long long)world * (long long)(Pf + Pb);
        const int lw = payload_lw(desc, D);
        if (da_raw) LMOE_CUDA_CHECK(cudaMemsetAsync(da_raw, 0, (size_t)H * 4, st));
        for (int r = 0; r < world; ++r) {
            int r0, len;
            slice(r, r0, len);
            LMOE_CUDA_CHECK(lmoe_dev::launch_rank_combine(dim3((D * D + 255) / 256, BH), st, fgath,
                                                          (int)payload_floats(desc, D), BH, r, D, D, 0, lw, M0,
                                                          nullptr));
            LMOE_CUDA_CHECK(lmoe_dev::launch_rank_combine_rev(bgath, (int)bwd_payload_floats(desc, D), BH, r, world,
                                                              D, D, lw, Xin, st));
            g_launch_count += 2;
            const int rc = lmoe_lsm_bwd(desc, B, len, H, D, dtype, at(q, r0, esz), at(k, r0, esz), at(v, r0, esz),
                                        at(a_pre, r0, esz), b_pre ? b_pre + (size_t)r0 * H : nullptr, a_raw, M0,
                                        at(dO, r0, esz), Xin, atw(dq, r0, esz), atw(dk, r0, esz), atw(dv, r0, esz),
                                        atw(da_pre, r0, esz), db_pre ? db_pre + (size_t)r0 * H : nullptr,
                                        da_raw ? dar : nullptr, r == 0 ? dM0 : nullptr, ws + w.off_bws, w.bws,
                                        stream);
            if (rc != LMOE_OK) throw Error(rc, lmoe_last_error());
            if (da_raw)
                LMOE_CUDA_CHECK(lmoe_dev::launch_norm_helpers(2, false, da_raw, dar, nullptr, nullptr, nullptr, nullptr,
                                                              1, H, nullptr, st));
        }
    });
}

// ------------------------------------------------------------- packed documents (varlen)
// model_forward (model.hpp:374-405) runs the mixer once per document of a PackedBatch
// (model.hpp:86-121): the state starts from zero at every boundary.  Each document is a
// dense row range of the packed [1, T, H, D] tensors, so the TMA bounds of its views clip
// exactly at the document end.  cu_seqlens is a HOST array of n_docs + 1 ascending offsets
// from 0 to T (PackedBatch::boundaries).
namespace lmoe_host {
static void check_bounds(const int* cu, int n_docs, int T) {
    if (!cu || n_docs < 1 || cu[0] != 0 || cu[n_docs] != T)
        throw Error(LMOE_ERR_ARG, "PackedBatch: boundaries must run from 0 to total length");
    for (int i = 1; i <= n_docs; ++i)
        if (cu[i] <= cu[i - 1]) throw Error(LMOE_ERR_ARG, "PackedBatch: boundaries must be strictly ascending");
}
static int max_doc(const int* cu, int n_docs) {
    int m = 0;
    for (int i = 0; i < n_docs; ++i) m = std::max(m, cu[i + 1] - cu[i]);
    return m;
}
}  // namespace lmoe_host

extern "C" size_t lmoe_lsm_varlen_workspace_size(const lmoe_lsm_desc* desc, int T, const int* cu_seqlens,
                                                 int n_docs, int H, int D, lmoe_dtype dtype, int backward) {
    if (!desc || T < 1 || !cu_seqlens || n_docs < 1 || H < 1 || D < 1) return 0;
    size_t m = 0;
    for (int i = 0; i < n_docs; ++i) {
        const int len = cu_seqlens[i + 1] - cu_seqlens[i];
        if (len < 1) return 0;
        m = std::max(m, backward ? lmoe_lsm_bwd_workspace_size(desc, 1, len, H, D, dtype)
                                 : plan_lsm(1, len, H, D).total);
    }
    return m;
}

extern "C" int lmoe_lsm_fwd_varlen(const lmoe_lsm_desc* desc, int T, const int* cu_seqlens, int n_docs, int H,
                                   int D, lmoe_dtype dtype, const void* q, const void* k, const void* v,
                                   const void* a_pre, const float* b_pre, const float* a_raw, void* o,
                                   float* M_out, void* workspace, size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        validate(desc, 1, T, H, D, dtype, q, k, v, o);
        check_bounds(cu_seqlens, n_docs, T);
        const size_t esz = dtype == LMOE_BF16 ? 2 : 4;
        const size_t row = (size_t)H * D * esz;
        for (int i = 0; i < n_docs; ++i) {
            const int r0 = cu_seqlens[i], len = cu_seqlens[i + 1] - r0;
            auto at = [&](const void* p) -> const void* { return p ? static_cast<const uint8_t*>(p) + r0 * row : nullptr; };
            const int rc = lmoe_lsm_fwd(desc, 1, len, H, D, dtype, at(q), at(k), at(v), at(a_pre),
                                        b_pre ? b_pre + (size_t)r0 * H : nullptr, a_raw, nullptr, nullptr,
                                        static_cast<uint8_t*>(o) + r0 * row,
                                        M_out ? M_out + (size_t)i * H * D * D : nullptr, nullptr, workspace,
                                        workspace_bytes, stream);
            if (rc != LMOE_OK) throw Error(rc, lmoe_last_error());
        }
    });
}

extern "C" int lmoe_lsm_bwd_varlen(const lmoe_lsm_desc* desc, int T, const int* cu_seqlens, int n_docs, int H,
                                   int D, lmoe_dtype dtype, const void* q, const void* k, const void* v,
                                   const void* a_pre, const float* b_pre, const float* a_raw, const void* dO,
                                   void* dq, void* dk, void* dv, void* da_pre, float* db_pre, float* da_raw,
                                   void* workspace, size_t workspace_bytes, lmoe_stream_t stream) {
    return guarded([&]() {
        validate(desc, 1, T, H, D, dtype, q, k, v, dO);
        check_bounds(cu_seqlens, n_docs, T);
        const size_t esz = dtype == LMOE_BF16 ? 2 : 4;
        const size_t row = (size_t)H * D * esz;
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        // da_raw sums over documents: each document's contribution lands in a scratch slot
        // after the largest document's workspace, then accumulates
        const size_t need = lmoe_lsm_varlen_workspace_size(desc, T, cu_seqlens, n_docs, H, D, dtype, 1);
        float* dar = nullptr;
        if (da_raw) {
            if (!workspace || workspace_bytes < align_up(need, 256) + (size_t)H * 4)
                throw Error(LMOE_ERR_ARG, "lmoe_lsm_bwd_varlen: workspace too small");
            dar = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + align_up(need, 256));
            LMOE_CUDA_CHECK(cudaMemsetAsync(da_raw, 0, (size_t)H * 4, st));
        }
        for (int i = 0; i < n_docs; ++i) {
            const int r0 = cu_seqlens[i], len = cu_seqlens[i + 1] - r0;
            auto at = [&](const void* p) -> const void* { return p ? static_cast<const uint8_t*>(p) + r0 * row : nullptr; };
            auto atw = [&](void* p) -> void* { return p ? static_cast<uint8_t*>(p) + r0 * row : nullptr; };
            const int rc = lmoe_lsm_bwd(desc, 1, len, H, D, dtype, at(q), at(k), at(v), at(a_pre),
                                        b_pre ? b_pre + (size_t)r0 * H : nullptr, a_raw, nullptr, at(dO), nullptr,
                                        atw(dq), atw(dk), atw(dv), atw(da_pre),
                                        db_pre ? db_pre + (size_t)r0 * H : nullptr, dar, nullptr, workspace, need,
                                        stream);
            if (rc != LMOE_OK) throw Error(rc, lmoe_last_error());
            if (da_raw)
                LMOE_CUDA_CHECK(lmoe_dev::launch_norm_helpers(2, false, da_raw, dar, nullptr, nullptr, nullptr, nullptr,
                                                              1, H, nullptr, st));
        }
    });
}
