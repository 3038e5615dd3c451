// context.h -- sd_ctx: one device, its resident geometry (per-kind
// primitive records grouped into (kind, polynomial) segments), weight
// table, tree and scratch. Internal to libsdgpu.so.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/sdgpu.h"
#include "exact.h"
#include "weights_host.h"

namespace sdgpu {

void set_error(const std::string& msg);

struct CudaError {
    cudaError_t code;
    std::string where;
};
void check_cuda(cudaError_t e, const char* where);  // throws CudaError

// A CUDA event released on every exit path (check_cuda throws).
struct ScopedEvent {
    cudaEvent_t e = nullptr;
    explicit ScopedEvent(unsigned flags = cudaEventDefault) {
        check_cuda(cudaEventCreateWithFlags(&e, flags), "cudaEventCreate");
    }
    ~ScopedEvent() {
        if (e) cudaEventDestroy(e);
    }
    ScopedEvent(const ScopedEvent&) = delete;
    ScopedEvent& operator=(const ScopedEvent&) = delete;
    operator cudaEvent_t() const { return e; }
};

// Grow-only device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    void* ensure(size_t n) {
        if (n > bytes) {
            release();
            check_cuda(cudaMalloc(&p, n ? n : 16), "cudaMalloc");
            bytes = n ? n : 16;
        }
        return p;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// A run of primitives of one kind sharing one weight polynomial
// (poly = -1: unit weight).
struct Segment {
    int kind;
    int poly;
    int64_t offset;  // first record in the kind's record array
    int64_t count;
    int64_t tile0;   // first tile box of the segment in the kind's box array
};

// Tree in traversal layout (pre-order ids == reference ids).
//   box[2 * id + 0] = (lo.xyz, diameter rounded to T)
//   box[2 * id + 1] = (hi.xyz, link) with link = right child id, or
//                     -(leaf slot + 1) on leaves
//   count[id]       = n_B;  diam64[id] = reference fp64 diameter
//   leaf slot s     -> leafrec[s * 24] unified record, leafmeta[s] =
//                      (kind | (poly + 1) << 2)
struct DeviceTree {
    int64_t nodes = 0;
    int64_t leaves = 0;
    int depth = 0;
    bool exact_boxes = true;
    DevBuf box, pairs, count, lgcount, diam64, leafrec, leafmeta;
    float contact_rc2 = -1.f;  // K3C search radius^2 (bvh.cu launch_contact_search); < 0: not computed
    int split_k = -1;         // depth of the cached split tables
    int64_t split_count = 0;  // slots at that depth
    DevBuf split_meta, split_path;  // see split_tables (bvh.cu)
};

struct Ctx {
    int device = 0;
    int precision = SD_FP32;
    cudaStream_t stream = nullptr;       // library-owned stream for host-buffer calls
    cudaStream_t copy_stream = nullptr;  // H2D / D2H of pipelined host-buffer batches

    // geometry (vertices already rounded to float in SD_FP32)
    std::vector<double> xyz;
    std::vector<int32_t> sv;
    std::vector<uint8_t> kind;
    int64_t V = 0, N = 0;
    bool have_geom = false;

    // weights
    bool have_weights = false;
    double A = 1.0, sup_wtilde = 1.0;
    std::vector<double> edge_a, tri_stored;
    std::vector<int32_t> poly_index;
    // per-polynomial metadata of the reference WeightSet (valences, extrema,
    // residual) for the SDWT0001 cache: edge (v0, v1) + (sup, inf), triangle
    // (v, e) + (sup, inf, residual); valence 0 = unknown
    std::vector<int32_t> edge_val, tri_val;
    std::vector<double> edge_ext, tri_ext;

    // exact layout
    bool exact_ready = false;
    std::vector<Segment> segs;
    DevBuf rec[3];
    DevBuf tbox[3];   // per kind: 2 float4 per tile (lo.xyz, diagonal) (hi.xyz, 0)
    double scene_lo[3] = {0, 0, 0}, scene_hi[3] = {0, 0, 0};

    // tree (host copy in the reference layout + device traversal layout)
    bool have_tree = false;
    bool tree_trusted = false;  // built here (pre-order, complete): no validation pass
    std::vector<sd_bvh_node> tree;
    DeviceTree dtree;
    bool dtree_ready = false;

    // simplex queries (simplex.cu): fp64 traversal layout of the same tree
    // (when the context is SD_FP32), fp64 leaf geometry in tree order and
    // per-primitive geometry in index order; rebuilt after any geometry,
    // weight or tree change
    DeviceTree dtree64;
    DevBuf leafgeom, primgeom, primmeta, qgeom, qdim;
    bool sx_tree_ready = false, sx_prim_ready = false;

    // pipelined host-buffer batches (sd_query_points_async): two slots, each
    // with its own device copies of a batch's queries and outputs; H2D on
    // in_stream, evaluation on `stream`, D2H on out_stream
    struct AsyncSlot {
        DevBuf qd, d, g, c, gc, l, f, h;
        cudaEvent_t in = nullptr, done = nullptr, out = nullptr;
        int64_t ticket = -1;
    };
    AsyncSlot slots[2];
    cudaStream_t in_stream = nullptr, out_stream = nullptr;
    int64_t next_ticket = 0;

    // K3C (bvh.cu): side stream of the near-contact search, fork / join
    // events, hit list
    cudaStream_t aux_stream = nullptr;
    cudaEvent_t aux_fork = nullptr, aux_join = nullptr;
    DevBuf contact_hits;
    unsigned contact_cap = 0;

    // scratch
    DevBuf qd, qT, part, out_d, out_g, out_c, out_gc, out_l, out_f, out_h;
    DevBuf perm, keys, tmp, tmp2, counters, polys, flag, qbox, aos;
    int64_t last_launches = 0;

    // sd_set_exact_pruning: 0 = every pair evaluated (the reference's sum),
    // > 0 = K1 skips tiles whose terms are below 2^-bits of the query's sum
    double exact_prune_bits = 0.0;

    // kernel timing (sd_set_kernel_timing): one event pair on the launching
    // stream around the dominant compute launches of every query call (the
    // exact segment launches, or the tree traversal), read back and recycled
    // by sd_kernel_times
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pairs;
    cudaEvent_t take_event() {
        cudaEvent_t e = nullptr;
        if (!ev_pool.empty()) {
            e = ev_pool.back();
            ev_pool.pop_back();
        } else {
            check_cuda(cudaEventCreate(&e), "cudaEventCreate");
        }
        return e;
    }
};

// Event pair around the dominant launches of one call (no-op unless the
// context's kernel timing is on).
struct KernelTimer {
    Ctx& c;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    KernelTimer(Ctx& ctx, cudaStream_t s) : c(ctx), st(s) {
        if (c.timing) {
            a = c.take_event();
            check_cuda(cudaEventRecord(a, st), "cudaEventRecord");
        }
    }
    void stop() {
        if (!a) return;
        cudaEvent_t b = c.take_event();
        check_cuda(cudaEventRecord(b, st), "cudaEventRecord");
        c.ev_pairs.emplace_back(a, b);
        a = nullptr;
    }
};

// Host helpers shared by api.cu / bvh.cu
template <class T>
Phys<T> make_phys(const Ctx& c, const sd_params& p);
template <class T>
Poly<T> make_poly(const Ctx& c, int kind, int poly, const sd_params& p);
bool poly_certified_positive(const Ctx& c, int kind, int poly);
template <class T>
void build_record(const Ctx& c, int64_t prim, T* out);  // rec_size(kind) values

template <class T>
const int64_t* sort_queries(Ctx& c, const T* q, int64_t Q, const double lo[3], const double hi[3], cudaStream_t st,
                            int64_t& launches, bool union_hilbert);  // Hilbert over box + query box, or Morton over box

// Tree entry points (bvh.cu)
void tree_upload(Ctx& c);  // host reference layout -> DeviceTree
void tree_upload64(Ctx& c, DeviceTree& t);  // same, fp64 records
void query_batch_f64(Ctx& c, const double* q, int64_t Q, const sd_params& p, int mode, const FinalizeOut& out,
                     cudaStream_t st);  // api.cu
void render_impl(Ctx& c, const sd_params& p, int mode, const sd_render_config& cfg, uint8_t* rgb, double* hit_t,
                 int64_t* stats, double* seconds);  // callers.cu
void grid_impl(Ctx& c, const sd_params& p, int mode, int n, double* d_hat, int64_t* leaves, int64_t* far,
               double* seconds);  // callers.cu
void simplex_query(Ctx& c, const double* corners, const int32_t* dims, int64_t Q, const sd_params& p, int mode,
                   const FinalizeOut& out, cudaStream_t st);
void split_tables(Ctx& c, DeviceTree& t, int k);  // nodes at depth k of c.tree
void tree_build_median_host(Ctx& c);  // bvh.cu, single-threaded restatement
void tree_build_median_gpu(Ctx& c);   // median.cu, same tree on the device
void tree_build_lbvh(Ctx& c);
WeightAssignment gpu_weight_assignment(Ctx& c);  // adjacency.cu
template <class T>
void tree_query(Ctx& c, const T* q, int64_t Q, const sd_params& p, const FinalizeOut& out, cudaStream_t st);

}  // namespace sdgpu

struct sd_ctx : sdgpu::Ctx {};
