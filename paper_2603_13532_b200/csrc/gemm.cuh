// gemm.cuh — grouped, batched, split-K fp64 GEMM on DMMA tensor cores (sm_100a).
//
// One launch covers many independent GEMMs ("groups"), each optionally strided-
// batched and split along K.  All stacked sketch contractions of the KRP sum are
// expressed through it (SURVEY.md §2.1 stages A, C, E, F, G-TTM, H):
//   C(M×N) = alpha · op(A) · op(B) + beta · C, column-major.
// Layouts (the three the pipeline needs):
//   TN : A stored K×M (k contiguous), B stored K×N (k contiguous)
//   NN : A stored M×K (m contiguous), B stored K×N (k contiguous)
//   NT : A stored M×K (m contiguous), B stored N×K (n contiguous)
// Split-K partials go to a workspace and are summed in split order by a second
// kernel, so results are deterministic run to run.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

#include "runtime.hpp"

namespace ts {

enum class Layout { TN, NN, NT };

struct GemmDesc {
    const double* A;
    const double* B;
    double* C;
    double* ws;  // split-K workspace [batch][splits][M*N] (only when splits > 1)
    int64_t lda, ldb, ldc;
    int64_t sA, sB, sC;  // batch strides (elements)
    int M, N, K, batch;
    int splits, tiles_m, tiles_n, k_per_split;
    double alpha, beta;
    int64_t unit_begin;  // first CTA unit of this group
};

// Host-side description before tiling decisions.
struct GemmProblem {
    const double* A;
    const double* B;
    double* C;
    int64_t lda, ldb, ldc;
    int64_t sA = 0, sB = 0, sC = 0;
    int M, N, K, batch = 1;
    double alpha = 1.0, beta = 0.0;
};

// Plans tiles/splits, uploads descriptors and launches the grouped GEMM (+ the
// split-K reduction when needed) on the scratch's stream.  `scratch` provides device memory
// for descriptors and split-K partials.  Returns the number of kernels launched.
// TMA + mbarrier warp-specialised path (gemm_tma.cu) for TN / NT problems with
// 16-byte aligned operands, even leading dimensions and batch 1.  Returns false
// without launching anything when the problems do not qualify.
bool launch_tma_gemm(Layout layout, const std::vector<GemmProblem>& probs, CallScratch& sc, int num_sms,
                     int* launched);
bool tma_gemm_enabled();

int launch_grouped_gemm(Layout layout, const std::vector<GemmProblem>& probs, CallScratch& scratch,
                        int num_sms);

}  // namespace ts
