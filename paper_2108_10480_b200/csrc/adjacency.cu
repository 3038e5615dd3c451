// adjacency.cu -- GPU precompute of the WeightSet assignment:
// build_adjacency (mesh.hpp:163-183) and the assignment half of
// build_weight_set (weights.hpp:589-621), which the reference runs as a
// single-threaded hash-map pass (seconds at cfg4/5 scale).
//
//   vertex valence   = number of incident non-point simplices (atomics)
//   edge valence     = number of edges / triangles containing the undirected
//                      edge: all edge keys sorted (CUB), counts found by
//                      binary search
//   per simplex key  = edge: (valence(v0), valence(v1)) in corner order;
//                      triangle: (max vertex valence, max edge valence)
//   polynomial ids   = distinct keys numbered in first-occurrence order
//                      (stable sort of (key, index), first index per run),
//                      edges and triangles numbered separately
//
// The polynomials themselves (closed-form edges; the triangle LP, once per
// distinct (v, e)) are built on the host from the distinct keys.
#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "context.h"
#include "weights_host.h"

namespace sdgpu {

namespace {

__device__ __forceinline__ uint64_t ekey(int32_t a, int32_t b) {
    if (a > b) {
        const int32_t t = a;
        a = b;
        b = t;
    }
    return (uint64_t(uint32_t(a)) << 32) | uint32_t(b);
}

__global__ void vertex_valence(const int32_t* __restrict__ sv, const uint8_t* __restrict__ kind, int64_t n,
                               int32_t* val) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int nv = kind[i] + 1;
    if (nv > 1)
        for (int a = 0; a < nv; ++a) atomicAdd(val + sv[3 * i + a], 1);
}

__global__ void edge_counts_per_simplex(const uint8_t* __restrict__ kind, int64_t n, int32_t* cnt) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    cnt[i] = kind[i] == 1 ? 1 : (kind[i] == 2 ? 3 : 0);
}

__global__ void emit_edge_keys(const int32_t* __restrict__ sv, const uint8_t* __restrict__ kind,
                               const int32_t* __restrict__ off, int64_t n, uint64_t* keys) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t* s = sv + 3 * i;
    uint64_t* k = keys + off[i];
    if (kind[i] == 1) {
        k[0] = ekey(s[0], s[1]);
    } else if (kind[i] == 2) {
        k[0] = ekey(s[0], s[1]);
        k[1] = ekey(s[1], s[2]);
        k[2] = ekey(s[2], s[0]);
    }
}

__device__ __forceinline__ int32_t count_key(const uint64_t* __restrict__ sorted, int64_t m, uint64_t key) {
    int64_t lo = 0, hi = m;  // lower bound
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (sorted[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    int64_t a = lo, b = m;  // upper bound
    while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (sorted[mid] <= key) a = mid + 1;
        else b = mid;
    }
    return int32_t(a - lo);
}

// key layout: kind (2 bits) << 62 | first << 31 | second; points: all ones
__global__ void simplex_keys(const int32_t* __restrict__ sv, const uint8_t* __restrict__ kind, int64_t n,
                             const int32_t* __restrict__ val, const uint64_t* __restrict__ sorted_edges, int64_t m,
                             uint64_t* keys, int64_t* idx) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t* s = sv + 3 * i;
    uint64_t k = ~0ull;
    if (kind[i] == 1) {
        k = (1ull << 62) | (uint64_t(uint32_t(val[s[0]])) << 31) | uint64_t(uint32_t(val[s[1]]));
    } else if (kind[i] == 2) {
        const int32_t v = max(val[s[0]], max(val[s[1]], val[s[2]]));
        const int32_t e = max(count_key(sorted_edges, m, ekey(s[0], s[1])),
                              max(count_key(sorted_edges, m, ekey(s[1], s[2])),
                                  count_key(sorted_edges, m, ekey(s[2], s[0]))));
        k = (2ull << 62) | (uint64_t(uint32_t(v)) << 31) | uint64_t(uint32_t(e));
    }
    keys[i] = k;
    idx[i] = i;
}

// first index of each run of equal keys (stable sort: the run's first element)
__global__ void run_firsts(const int64_t* __restrict__ sorted_idx, const int32_t* __restrict__ run_off, int runs,
                           int64_t* first) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < runs) first[r] = sorted_idx[run_off[r]];
}

__global__ void assign_ids(const uint64_t* __restrict__ keys, int64_t n, const uint64_t* __restrict__ ukeys,
                           const int32_t* __restrict__ uid, int runs, int32_t* poly_index) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t k = keys[i];
    int lo = 0, hi = runs;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ukeys[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    poly_index[i] = uid[lo];
}

}  // namespace

WeightAssignment gpu_weight_assignment(Ctx& c) {
    WeightAssignment out;
    const int64_t n = c.N;
    out.poly_index.assign(size_t(n), -1);
    if (n == 0) return out;
    cudaStream_t st = c.stream;
    const unsigned B = 256;
    const unsigned G = unsigned((n + B - 1) / B);
    DevBuf d_sv, d_kind, d_val, d_cnt, d_off, d_ek, d_keys, d_idx, d_tmp, d_runs, d_rcnt, d_nruns, d_first, d_map,
        d_pi;
    int32_t* sv = static_cast<int32_t*>(d_sv.ensure(c.sv.size() * sizeof(int32_t)));
    uint8_t* kind = static_cast<uint8_t*>(d_kind.ensure(c.kind.size()));
    int32_t* val = static_cast<int32_t*>(d_val.ensure(size_t(std::max<int64_t>(c.V, 1)) * sizeof(int32_t)));
    check_cuda(cudaMemcpyAsync(sv, c.sv.data(), c.sv.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st), "H2D");
    check_cuda(cudaMemcpyAsync(kind, c.kind.data(), c.kind.size(), cudaMemcpyHostToDevice, st), "H2D");
    check_cuda(cudaMemsetAsync(val, 0, size_t(std::max<int64_t>(c.V, 1)) * sizeof(int32_t), st), "memset");
    vertex_valence<<<G, B, 0, st>>>(sv, kind, n, val);
    check_cuda(cudaGetLastError(), "vertex valence");

    // all edge keys, sorted
    int32_t* cnt = static_cast<int32_t*>(d_cnt.ensure(size_t(n) * sizeof(int32_t)));
    int32_t* off = static_cast<int32_t*>(d_off.ensure(size_t(n + 1) * sizeof(int32_t)));
    edge_counts_per_simplex<<<G, B, 0, st>>>(kind, n, cnt);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, int(n), st);
    check_cuda(cub::DeviceScan::ExclusiveSum(d_tmp.ensure(tb), tb, cnt, off, int(n), st), "scan");
    int32_t last_off = 0, last_cnt = 0;
    check_cuda(cudaMemcpyAsync(&last_off, off + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaMemcpyAsync(&last_cnt, cnt + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaStreamSynchronize(st), "adjacency");
    const int64_t m = int64_t(last_off) + last_cnt;
    uint64_t* ek = static_cast<uint64_t*>(d_ek.ensure(size_t(std::max<int64_t>(m, 1)) * 2 * sizeof(uint64_t)));
    emit_edge_keys<<<G, B, 0, st>>>(sv, kind, off, n, ek);
    if (m > 0) {
        tb = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb, ek, ek + m, int(m), 0, 62, st);
        check_cuda(cub::DeviceRadixSort::SortKeys(d_tmp.ensure(tb), tb, ek, ek + m, int(m), 0, 62, st),
                   "sort edge keys");
    }
    const uint64_t* sorted_edges = ek + m;

    // per-simplex keys, stable-sorted with their index; runs -> distinct keys
    uint64_t* keys = static_cast<uint64_t*>(d_keys.ensure(size_t(n) * 2 * sizeof(uint64_t)));
    int64_t* idx = static_cast<int64_t*>(d_idx.ensure(size_t(n) * 2 * sizeof(int64_t)));
    simplex_keys<<<G, B, 0, st>>>(sv, kind, n, val, sorted_edges, m, keys, idx);
    check_cuda(cudaGetLastError(), "simplex keys");
    tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys + n, idx, idx + n, int(n), 0, 64, st);
    check_cuda(cub::DeviceRadixSort::SortPairs(d_tmp.ensure(tb), tb, keys, keys + n, idx, idx + n, int(n), 0, 64, st),
               "sort simplex keys");
    uint64_t* runs = static_cast<uint64_t*>(d_runs.ensure(size_t(n) * sizeof(uint64_t)));
    int32_t* rcnt = static_cast<int32_t*>(d_rcnt.ensure(size_t(n) * sizeof(int32_t)));
    int32_t* nruns = static_cast<int32_t*>(d_nruns.ensure(sizeof(int32_t)));
    tb = 0;
    cub::DeviceRunLengthEncode::Encode(nullptr, tb, keys + n, runs, rcnt, nruns, int(n), st);
    check_cuda(cub::DeviceRunLengthEncode::Encode(d_tmp.ensure(tb), tb, keys + n, runs, rcnt, nruns, int(n), st),
               "run-length encode");
    int32_t R = 0;
    check_cuda(cudaMemcpyAsync(&R, nruns, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaStreamSynchronize(st), "adjacency");
    // run offsets (scan of the counts) -> first index of every run
    int32_t* roff = static_cast<int32_t*>(d_off.ensure(size_t(n + 1) * sizeof(int32_t)));
    tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, rcnt, roff, R, st);
    check_cuda(cub::DeviceScan::ExclusiveSum(d_tmp.ensure(tb), tb, rcnt, roff, R, st), "scan");
    int64_t* first = static_cast<int64_t*>(d_first.ensure(size_t(R) * sizeof(int64_t)));
    run_firsts<<<unsigned((R + 255) / 256), 256, 0, st>>>(idx + n, roff, R, first);
    std::vector<uint64_t> ukeys(static_cast<size_t>(R));
    std::vector<int64_t> ufirst(static_cast<size_t>(R));
    check_cuda(cudaMemcpyAsync(ukeys.data(), runs, size_t(R) * sizeof(uint64_t), cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaMemcpyAsync(ufirst.data(), first, size_t(R) * sizeof(int64_t), cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaStreamSynchronize(st), "adjacency");

    // first-occurrence numbering, edges and triangles separately
    std::vector<int> order(static_cast<size_t>(R));
    for (int r = 0; r < R; ++r) order[r] = r;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return ufirst[x] < ufirst[y]; });
    std::vector<int32_t> uid(static_cast<size_t>(R), -1);
    for (int r : order) {
        const uint64_t k = ukeys[r];
        if (k == ~0ull) continue;  // points
        const int kd = int(k >> 62);
        const int32_t a = int32_t((k >> 31) & 0x7fffffffull), b = int32_t(k & 0x7fffffffull);
        if (kd == 1) {
            uid[r] = int32_t(out.edge_keys.size());
            out.edge_keys.push_back({a, b});
        } else {
            uid[r] = int32_t(out.tri_keys.size());
            out.tri_keys.push_back({a, b});
        }
    }
    int32_t* map = static_cast<int32_t*>(d_map.ensure(size_t(R) * sizeof(int32_t)));
    int32_t* pi = static_cast<int32_t*>(d_pi.ensure(size_t(n) * sizeof(int32_t)));
    check_cuda(cudaMemcpyAsync(map, uid.data(), size_t(R) * sizeof(int32_t), cudaMemcpyHostToDevice, st), "H2D");
    assign_ids<<<G, B, 0, st>>>(keys, n, runs, map, R, pi);
    check_cuda(cudaGetLastError(), "assign ids");
    check_cuda(cudaMemcpyAsync(out.poly_index.data(), pi, size_t(n) * sizeof(int32_t), cudaMemcpyDeviceToHost, st),
               "D2H");
    check_cuda(cudaStreamSynchronize(st), "adjacency");
    return out;
}

}  // namespace sdgpu
