// Host interface of the device k-means (kmeans.cu).
#pragma once

#include <vector>

#include "engine.h"

namespace dqtg {

// One clustering problem = one approx_kmeans call (quantize.cpp:256-325) after
// the histogram: n distinct ascending keys with mixed weights, k centres.
struct KProblem {
    const double* pts;
    const double* w;
    int n, k;
    uint64_t seed;  // restart t uses seed + t (quantize.cpp:310)
    int skip;       // problem resolved elsewhere (e.g. distinct-value shortcut)
    int slot;       // codebook output slot
    double* scratch;
    size_t scratch_stride;
    double* centers;  // [restarts][k]
    double* loss;     // [restarts]
};

void run_kmeans(Engine& e, std::vector<KProblem>& probs, float* cb_out, int cb_stride,
                uint32_t* cb_len_dev);
void compact_keys(Engine& e, const unsigned long long* hist, int64_t hs_stride, int64_t HS,
                  const double* key, double sigma, int nprob, double* pts,
                  unsigned long long* cnt, double* w, int64_t out_stride, int* n_keys);

}  // namespace dqtg
