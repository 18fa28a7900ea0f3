// lsm_host.cu -- host orchestration of the LSM forward: argument validation with the
// reference's error texts, segment planning, workspace carving, TMA descriptors, launches.
#include <cmath>
#include <vector>

#include "common.h"
#include "lsm_fwd.cu"

namespace lmoe_host {

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
        default: return -1;
    }
}

struct LsmPlan {
    int seg_len = 0, nseg = 0;
    size_t off_S = 0, off_z = 0, off_logD = 0, off_Min = 0, off_zin = 0, off_err = 0, total = 0;
};

// Segment length: a multiple of the 128-token tile chosen so the B*H*nseg CTAs of the
// segment-parallel passes fill whole waves of the SMs (one CTA per SM).
static LsmPlan plan_lsm(int B, int N, int H, int D) {
    LsmPlan pl;
    const int C = lmoe_dev::kC;
    const int chunks = (N + C - 1) / C;
    const long long heads = (long long)B * H;
    const int sms = num_sms();
    double best = -1.0;
    for (int waves = 1; waves <= 12; ++waves) {
        long long target = (long long)sms * waves;
        int seg_chunks = (int)std::max<long long>(1, (heads * chunks + target - 1) / target);
        seg_chunks = std::min(seg_chunks, chunks);
        int nseg = (chunks + seg_chunks - 1) / seg_chunks;
        long long ctas = heads * nseg;
        long long w = (ctas + sms - 1) / sms;
        double eff = (double)(heads * chunks) / (double)(w * sms * seg_chunks);
        // prefer fuller waves, then fewer segments (less combine traffic)
        double score = eff - 0.002 * waves;
        if (score > best) {
            best = score;
            pl.seg_len = seg_chunks * C;
            pl.nseg = nseg;
        }
    }
    const size_t heads_nseg = (size_t)heads * pl.nseg;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    pl.off_S = take(heads_nseg * D * D * 4);
    pl.off_z = take(heads_nseg * D * 4);
    pl.off_logD = take(heads_nseg * 4);
    pl.off_Min = take(heads_nseg * D * D * 4);
    pl.off_zin = take(heads_nseg * D * 4);
    pl.off_err = take(64);
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

template <typename T>
static void launch_lsm(const lmoe_lsm_desc* d, int B, int N, int H, lmoe_dtype dt, const void* q,
                       const void* k, const void* v, const float* b_pre, const float* a_raw,
                       const float* M0, const float* z0, void* o, float* M_out, float* z_out,
                       uint8_t* ws, const LsmPlan& pl, cudaStream_t st) {
    using TT = lmoe_dev::TileTraits<T>;
    constexpr int D = TT::D;
    const CUtensorMapDataType tdt =
        sizeof(T) == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const CUtensorMap tq = make_tmap_4d(q, tdt, sizeof(T), D, H, N, B, TT::EPB, lmoe_dev::kC);
    const CUtensorMap tk = make_tmap_4d(k, tdt, sizeof(T), D, H, N, B, TT::EPB, lmoe_dev::kC);
    const CUtensorMap tv = make_tmap_4d(v, tdt, sizeof(T), D, H, N, B, TT::EPB, lmoe_dev::kC);
    const CUtensorMap to = make_tmap_4d(o, tdt, sizeof(T), D, H, N, B, TT::EPB, lmoe_dev::kC);

    lmoe_dev::LsmFwdParams p{};
    p.B = B; p.N = N; p.H = H;
    p.seg_len = pl.seg_len;
    p.nseg = pl.nseg;
    p.decay = device_decay_mode(d->instance);
    p.fm = d->feature_map;
    p.norm = d->use_normalizer;
    p.mamba2_keff = d->instance == LMOE_MAMBA2;
    p.log_a = p.decay == lmoe_dev::kDecayConst ? logf(d->scalar_decay) : 0.f;
    p.b_pre = b_pre;
    p.a_raw = a_raw;
    p.Sseg = reinterpret_cast<float*>(ws + pl.off_S);
    p.zseg = reinterpret_cast<float*>(ws + pl.off_z);
    p.logDseg = reinterpret_cast<float*>(ws + pl.off_logD);
    p.Min = reinterpret_cast<const float*>(ws + pl.off_Min);
    p.zin = reinterpret_cast<const float*>(ws + pl.off_zin);
    p.err = reinterpret_cast<int*>(ws + pl.off_err);
    if (p.decay == lmoe_dev::kDecayTokenScalar && (!b_pre || !a_raw))
        throw Error(LMOE_ERR_ARG, "lmoe_lsm_fwd: Mamba2 needs b_pre and a_raw");

    static bool attr_done[2] = {false, false};
    const int ai = sizeof(T) == 2 ? 0 : 1;
    if (!attr_done[ai]) {
        LMOE_CUDA_CHECK(cudaFuncSetAttribute(lmoe_dev::lsm_state_pass<T>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             lmoe_dev::kStatePassSmem));
        LMOE_CUDA_CHECK(cudaFuncSetAttribute(lmoe_dev::lsm_output_pass<T>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             lmoe_dev::output_pass_smem<T>()));
        attr_done[ai] = true;
    }
    LMOE_CUDA_CHECK(cudaMemsetAsync(p.err, 0, 64, st));
    const dim3 grid(pl.nseg, H, B);
    lmoe_dev::lsm_state_pass<T><<<grid, lmoe_dev::kStatePassThreads, lmoe_dev::kStatePassSmem, st>>>(tk, tv, p);
    LMOE_CUDA_CHECK(cudaGetLastError());
    const int nel = D * D + (p.norm ? D : 0);
    lmoe_dev::lsm_seg_combine<<<dim3((nel + 255) / 256, B * H), 256, 0, st>>>(
        p.Sseg, p.zseg, p.logDseg, M0, z0, const_cast<float*>(p.Min), const_cast<float*>(p.zin),
        M_out, z_out, pl.nseg, D, D, p.norm, p.err);
    LMOE_CUDA_CHECK(cudaGetLastError());
    lmoe_dev::lsm_output_pass<T><<<grid, lmoe_dev::kOutputPassThreads, lmoe_dev::output_pass_smem<T>(), st>>>(
        tq, tk, tv, to, p);
    LMOE_CUDA_CHECK(cudaGetLastError());
    g_launch_count += 3;
    if (d->flags & LMOE_FLAG_CHECK) {
        int err[2] = {0, 0};
        LMOE_CUDA_CHECK(cudaMemcpyAsync(err, p.err, sizeof(err), cudaMemcpyDeviceToHost, st));
        LMOE_CUDA_CHECK(cudaStreamSynchronize(st));
        if (err[0])
            throw Error(LMOE_ERR_DEGENERATE,
                        std::string("degenerate normalizer in instance ") + instance_name(d->instance));
        if (err[1])
            throw Error(LMOE_ERR_NONFINITE,
                        std::string("non-finite memory state in instance ") + instance_name(d->instance));
    }
    (void)dt;
}

}  // namespace lmoe_host

using namespace lmoe_host;

extern "C" size_t lmoe_lsm_fwd_workspace_size(const lmoe_lsm_desc* desc, int B, int N, int H,
                                              int D, lmoe_dtype dtype) {
    (void)desc; (void)dtype;
    if (B < 1 || N < 1 || H < 1 || D < 1) return 0;
    return plan_lsm(B, N, H, D).total;
}

extern "C" int lmoe_lsm_fwd_num_launches(const lmoe_lsm_desc* desc) {
    (void)desc;
    return 3;
}

extern "C" int lmoe_lsm_fwd(const lmoe_lsm_desc* desc, int B, int N, int H, int D,
                            lmoe_dtype dtype, const void* q, const void* k, const void* v,
                            const void* a_pre, const float* b_pre, const float* a_raw,
                            const float* M0, const float* z0, void* o, float* M_out,
                            float* z_out, void* workspace, size_t workspace_bytes,
                            lmoe_stream_t stream) {
    return guarded([&]() {
        validate(desc, B, N, H, D, dtype, q, k, v, o);
        (void)a_pre;
        const LsmPlan pl = plan_lsm(B, N, H, D);
        if (!workspace || workspace_bytes < pl.total)
            throw Error(LMOE_ERR_ARG, "lmoe_lsm_fwd: workspace too small (need " +
                                          std::to_string(pl.total) + " bytes)");
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        if (dtype == LMOE_BF16)
            launch_lsm<__nv_bfloat16>(desc, B, N, H, dtype, q, k, v, b_pre, a_raw, M0, z0, o,
                                      M_out, z_out, static_cast<uint8_t*>(workspace), pl, st);
        else
            launch_lsm<float>(desc, B, N, H, dtype, q, k, v, b_pre, a_raw, M0, z0, o, M_out,
                              z_out, static_cast<uint8_t*>(workspace), pl, st);
    });
}
