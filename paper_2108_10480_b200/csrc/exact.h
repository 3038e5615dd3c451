// exact.h -- host-side launch descriptors for the kernels (K1 exact, K3
// tree traversal, K4 epilogue). Internal to libsdgpu.so.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "pair.cuh"

namespace sdgpu {

template <class T>
struct ExactLaunch {
    int kind = 0;          // SD_POINT / SD_EDGE / SD_TRIANGLE
    bool has_poly = false; // false: unit weight (w = A^S)
    bool safe = false;     // polynomial certified positive: no 1e-300 floor selects
    const T* rec = nullptr;
    int64_t count = 0;     // primitives in the segment
    int64_t chunk = 0;     // primitives per split
    int splits = 1;
    // the split CTAs of a query block form one thread-block cluster and
    // merge their per-query totals over distributed shared memory: only
    // split 0's partial is written (splits <= 16)
    bool cluster = false;
    const T* q = nullptr;
    int64_t Q = 0;
    double* part = nullptr;  // [splits][5][Q] fp64 partial state
    int first = 1;
    Phys<T> ph{};
    Poly<T> poly{};
    const int64_t* perm = nullptr;  // sorted position -> query index (spatial order)
    const float4* tbox = nullptr;   // tile boxes of this segment (2 float4 per tile), or null
    T lwmax = T(0);                 // upper bound of log2 w over the segment (unit: 0, shift-relative)
    T lwspan = T(0);                // lwmax - lower bound of log2 w
    // > 0: pruned evaluation (sd_set_exact_pruning): a warp skips a tile when
    // every term of it is below 2^-prune of a lower bound of the query's sum
    float prune = 0.f;
};

template <class T>
cudaError_t launch_exact(const ExactLaunch<T>& L, cudaStream_t st);
template <class T>
int64_t exact_queries_per_cta(int kind);
int exact_tile_prims(int kind);  // primitives per staged tile (tile boxes use the same grid)
template <class T>
int exact_blocks_per_sm(int kind, bool has_poly, bool safe);  // resident CTAs per SM

// K4: merge `splits` partial states and finalise (smooth.hpp:147-159).
struct FinalizeOut {
    double* d_hat = nullptr;
    double* grad = nullptr;
    double* c = nullptr;
    double* grad_c = nullptr;
    int64_t* leaves = nullptr;
    int64_t* far_field = nullptr;
    uint64_t* hash = nullptr;
    // primitive-sharded exchange fused into the epilogue: when set, the
    // unshifted partials (c, grad_c) of query j go straight into the owner's
    // symmetric buffer peers[j / peer_qown] (slot peer_rank, SoA [4][qown])
    // instead of d_hat / grad / c / grad_c
    double* const* peers = nullptr;
    int peer_rank = 0;
    int64_t peer_qown = 0;
    // the batch's query points (context precision, input order): a query
    // with a NaN coordinate reports NaN d_hat / grad / c / grad_c, as the
    // reference's exp(NaN) does (the kernels mask NaN distances like
    // overflowed ones, so the NaN is restored here)
    const float* qf = nullptr;
    const double* qd = nullptr;
    // or, for sorted tree batches: the sorted Hilbert keys, 0xffffffff
    // marking a query with a NaN coordinate (query_morton*): read in sorted
    // order instead of the scattered re-read of the query
    const uint32_t* nan_keys = nullptr;
    // scratch of 4 doubles per query (sorted tree batches): K4 scatters
    // (d_hat, grad) as ONE 32-byte sector per query into it, and a
    // coalesced pass splits it into d_hat / grad (instead of partial-sector
    // scatters into both arrays)
    double* aos = nullptr;
    // query-sharded tree evaluation (sd_query_points_device_shard): only
    // this rank's chunks of pk_chunk 32-query packets of the sorted batch
    // (chunk j belongs to rank j % pk_world)
    int64_t pk_world = 1, pk_rank = 0, pk_chunk = 1;
};

// k-th packet of a rank's share (chunks of C packets dealt round robin)
__host__ __device__ __forceinline__ int64_t shard_packet(int64_t k, int64_t W, int64_t r, int64_t C) {
    return ((k / C) * W + r) * C + k % C;
}
// number of packets of the rank among npk
__host__ __device__ __forceinline__ int64_t shard_count(int64_t npk, int64_t W, int64_t r, int64_t C) {
    const int64_t full = npk / (C * W), rem = npk - full * C * W;
    const int64_t tail = rem - r * C;
    return full * C + (tail < 0 ? 0 : (tail > C ? C : tail));
}

cudaError_t launch_finalize(const double* part, int splits, int64_t Q, double alpha, double epsilon,
                            int64_t const_leaves, const int64_t* leaves_in, const int64_t* far_in,
                            const uint64_t* hash_in, const int64_t* perm, const FinalizeOut& out, cudaStream_t st);
cudaError_t launch_finalize_sums(const double* c, const double* grad_c, int64_t Q, double alpha, double epsilon,
                                 double* d_hat, double* grad, cudaStream_t st);

// Primitive-sharded exchange through peer memory (epilogue.cu).
cudaError_t launch_scatter_partials(const double* c, const double* grad_c, int64_t Q, double* const* peers, int rank,
                                    int64_t qown, cudaStream_t st);
cudaError_t launch_reduce_owned(const double* sbuf, int64_t qown, int64_t n, int world, double alpha, double epsilon,
                                double* d_hat, double* grad, cudaStream_t st);

// Mesh-to-mesh outer LogSumExp (smooth.hpp:237-254); vidx stride 1: point
// simplices, stride 3: corner lists (-1 padded).
cudaError_t launch_mesh_reduce(const double* d, const double* grad, int64_t n, const int32_t* vidx, int stride,
                               int64_t nv,
                               double alpha_q, double eps, double* work, size_t work_bytes, double* vg,
                               double* d_out, int64_t& launches, cudaStream_t st);
size_t mesh_reduce_work_bytes(int64_t n);

// Fills an empty-mesh result (+inf, zero gradient; smooth.hpp:151-155).
cudaError_t launch_empty_result(int64_t Q, const FinalizeOut& out, cudaStream_t st);

}  // namespace sdgpu
