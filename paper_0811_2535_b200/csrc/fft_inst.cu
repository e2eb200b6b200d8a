// fft_inst.cu -- instantiates the pass kernel for one FFT length F = 2^MOA_INST_LOGF.
// Compiled once per length (1..13) with -DMOA_INST_LOGF=<f>, in parallel.
#include "fft_pass.cuh"

#ifndef MOA_INST_LOGF
#error "compile with -DMOA_INST_LOGF=<1..13>"
#endif

#define MOA_CAT2(a, b) a##b
#define MOA_CAT(a, b) MOA_CAT2(a, b)

namespace moa {

static constexpr int kF = 1 << MOA_INST_LOGF;

template <int T>
static cudaError_t launch_t(const PassDesc &d, int64_t tiles, cudaStream_t s) {
    if constexpr (T * kF <= TF_MAX) return launch_one<kF, T>(d, tiles, s);
    return cudaErrorInvalidValue;
}

template <int T>
static cudaError_t prepare_t() {
    if constexpr (T * kF <= TF_MAX) return prepare_one<kF, T>();
    return cudaSuccess;
}

cudaError_t MOA_CAT(launch_pass_f, MOA_INST_LOGF)(int T, const PassDesc &d, int64_t tiles, cudaStream_t s) {
    switch (T) {
    case 1: return launch_t<1>(d, tiles, s);
    case 2: return launch_t<2>(d, tiles, s);
    case 4: return launch_t<4>(d, tiles, s);
    case 8: return launch_t<8>(d, tiles, s);
    case 16: return launch_t<16>(d, tiles, s);
    case 32: return launch_t<32>(d, tiles, s);
    case 64: return launch_t<64>(d, tiles, s);
    default: return cudaErrorInvalidValue;
    }
}

// row pass with bulk-tensor stores (ST = 4): F >= 256, 2T doubles per box row
cudaError_t MOA_CAT(launch_pass_tmast_f, MOA_INST_LOGF)(int T, const PassDesc &d, const CUtensorMap &omap,
                                                       int64_t tiles, cudaStream_t s) {
#define MOA_TMAST_CASE(TT)                                                                       \
    if (T == TT) {                                                                               \
        if constexpr (kF >= 256 && TT * kF <= TF_MAX) return launch_tmast<kF, TT>(d, omap, tiles, s); \
        return cudaErrorInvalidValue;                                                            \
    }
    MOA_TMAST_CASE(1)
    MOA_TMAST_CASE(2)
    MOA_TMAST_CASE(4)
    MOA_TMAST_CASE(8)
    MOA_TMAST_CASE(16)
#undef MOA_TMAST_CASE
    return cudaErrorInvalidValue;
}

#ifdef MOA_VARIANTS
// TMA-staged persistent variants: F >= 32, T*F <= 4096 (staging + exchange buffers fit)
template <int T, int SRC>
static constexpr bool tma_ok() {
    return kF >= 32 && T * kF <= 4096 && T * kF >= 256;
}

cudaError_t MOA_CAT(launch_pass_tma_f, MOA_INST_LOGF)(int T, int src, const PassDesc &d, const CUtensorMap &map,
                                                     int64_t tiles, int grid, cudaStream_t s) {
#define MOA_TMA_CASE(TT)                                                                   \
    if (T == TT) {                                                                         \
        if constexpr (tma_ok<TT, 1>()) {                                                   \
            if (src == 1) return launch_one_tma<kF, TT, 1>(d, map, tiles, grid, s);        \
            if (src == 2) return launch_one_tma<kF, TT, 2>(d, map, tiles, grid, s);        \
            if (src == 4) return launch_one_tpf<kF, TT, 4>(d, map, tiles, grid, s);        \
            if (src == 5) return launch_one_tpf<kF, TT, 5>(d, map, tiles, grid, s);        \
            if (src == 6) return launch_one_tma1<kF, TT, 6>(d, map, tiles, s);             \
            if (src == 7) return launch_one_tma1<kF, TT, 7>(d, map, tiles, s);             \
        }                                                                                  \
        return cudaErrorInvalidValue;                                                      \
    }
    MOA_TMA_CASE(1)
    MOA_TMA_CASE(2)
    MOA_TMA_CASE(4)
    MOA_TMA_CASE(8)
    MOA_TMA_CASE(16)
    MOA_TMA_CASE(32)
    MOA_TMA_CASE(64)
#undef MOA_TMA_CASE
    return cudaErrorInvalidValue;
}

int MOA_CAT(grid_pass_tma_f, MOA_INST_LOGF)(int T, int src) {
#define MOA_TMA_GRID(TT)                                                \
    if (T == TT) {                                                      \
        if constexpr (tma_ok<TT, 1>()) {                                \
            if (src == 1) return grid_one_tma<kF, TT, 1>();             \
            if (src == 2) return grid_one_tma<kF, TT, 2>();             \
            if (src == 4) return grid_one_tpf<kF, TT, 4>();             \
            if (src == 5) return grid_one_tpf<kF, TT, 5>();             \
            if (src == 6 || src == 7) return 1;                         \
        }                                                               \
        return 0;                                                       \
    }
    MOA_TMA_GRID(1)
    MOA_TMA_GRID(2)
    MOA_TMA_GRID(4)
    MOA_TMA_GRID(8)
    MOA_TMA_GRID(16)
    MOA_TMA_GRID(32)
    MOA_TMA_GRID(64)
#undef MOA_TMA_GRID
    return 0;
}

// prefetching persistent variant: F >= 32 (at least two stages)
cudaError_t MOA_CAT(launch_pass_pf_f, MOA_INST_LOGF)(int T, const PassDesc &d, int64_t tiles, int grid,
                                                    cudaStream_t s) {
#define MOA_PF_CASE(TT)                                                              \
    if (T == TT) {                                                                   \
        if constexpr (kF >= 32 && TT * kF <= TF_MAX) return launch_one_pf<kF, TT>(d, tiles, grid, s); \
        return cudaErrorInvalidValue;                                                \
    }
    MOA_PF_CASE(1)
    MOA_PF_CASE(2)
    MOA_PF_CASE(4)
    MOA_PF_CASE(8)
    MOA_PF_CASE(16)
    MOA_PF_CASE(32)
    MOA_PF_CASE(64)
#undef MOA_PF_CASE
    return cudaErrorInvalidValue;
}

int MOA_CAT(grid_pass_pf_f, MOA_INST_LOGF)(int T) {
#define MOA_PF_GRID(TT)                                                         \
    if (T == TT) {                                                              \
        if constexpr (kF >= 32 && TT * kF <= TF_MAX) return grid_one_pf<kF, TT>(); \
        return 0;                                                               \
    }
    MOA_PF_GRID(1)
    MOA_PF_GRID(2)
    MOA_PF_GRID(4)
    MOA_PF_GRID(8)
    MOA_PF_GRID(16)
    MOA_PF_GRID(32)
    MOA_PF_GRID(64)
#undef MOA_PF_GRID
    return 0;
}

#endif  // MOA_VARIANTS

cudaError_t MOA_CAT(prepare_pass_f, MOA_INST_LOGF)() {
    cudaError_t e;
    if ((e = prepare_t<1>()) != cudaSuccess) return e;
    if ((e = prepare_t<2>()) != cudaSuccess) return e;
    if ((e = prepare_t<4>()) != cudaSuccess) return e;
    if ((e = prepare_t<8>()) != cudaSuccess) return e;
    if ((e = prepare_t<16>()) != cudaSuccess) return e;
    if ((e = prepare_t<32>()) != cudaSuccess) return e;
    return prepare_t<64>();
}

}  // namespace moa
