// Slab-sharded ADMM-TV and Tikhonov over P ranks, one GPU per rank
// (BASELINE configs 3 and 4 "slab-decomposed across 1/2/4/8 B200").
//
// Decomposition.  Spatially, rank p owns the HR rows y in [p n/P, (p+1) n/P)
// of every plane (a y-slab: axis 3 stays whole, so the paired real axis-3
// transform is local).  Spectrally, after that r2c, the Hermitian half
// spectrum along axis 3 (planes f3 = 0..s/2) is partitioned by PLANE: the LR
// classes g3 are grouped in conjugate pairs {g3, -g3 mod sl}, and rank p owns
// every half-spectrum plane f3 whose class is in its pairs, with all rows f2.
// An alias set of the fold, rows (g2 + bc nl, g3 + bs sl), then lives on ONE
// rank: rows past the Nyquist plane are conj(row(-f2, s - f3)) of class -g3,
// which the same rank owns.  So the axis-2 passes and the axis-1 fold
// sandwich run locally, unchanged.
//
// Exchange = the kernels' own loads/stores over NVLink peer memory.  The
// axis-3 r2c stores each output plane straight into its owner's spectral
// buffer (this rank's rows of that plane are one contiguous run there); the
// inverse c2r pulls them back; the stencil reads its y halos (x rows -1 and
// n/P, dual row -1) from the neighbours' slabs in place.  Buffers are shared
// through CUDA IPC handles; each exchange point is a stream-ordered barrier
// (a one-word NCCL all-reduce).  Three barriers per ADMM-TV iteration, no
// packing passes and no staging copies; half of a full-spectrum exchange.
//
// Backends (vsr_comm): NCCL (one process per GPU; libnccl is loaded at run
// time), host callbacks (the caller's barrier / all-gather, e.g. gloo - the
// multi-process tests), and local (P virtual ranks in one process on one
// device, run stage by stage in stream order - no kernel ever waits on
// another).  Scalars are summed in rank order: deterministic for a given P.
//
// Reference: solvers.cpp:321-411 (admm_tv), :36-67 (TikhonovOperator).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/vsr.h"
#include "fft.cuh"
#include "fold.cuh"
#include "fused.cuh"
#include "host_util.cuh"
#include "tv.cuh"

using namespace vsr;
using namespace vsr_host;

namespace vsr_capi {
cudaStream_t stream_of(vsr_ctx* ctx);
int device_of(vsr_ctx* ctx);
int guard_call(const std::function<void()>& f);
void add_fft_counts(uint64_t forward, uint64_t inverse);
}  // namespace vsr_capi

namespace {

struct DevGuard {
    int prev = 0;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) VSR_CUDA(cudaSetDevice(dev));
    }
    ~DevGuard() {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != prev) cudaSetDevice(prev);
    }
};

// ------------------------------------------------------------------ NCCL
// Loaded at run time (the process's libnccl.so.2, e.g. torch's), so the
// library has no link-time NCCL dependency and a missing NCCL is a clean error.
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string why;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return a;
        }
        a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
        a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(h, "ncclCommInitRank");
        a.comm_destroy = (decltype(a.comm_destroy))dlsym(h, "ncclCommDestroy");
        a.all_reduce = (decltype(a.all_reduce))dlsym(h, "ncclAllReduce");
        a.all_gather = (decltype(a.all_gather))dlsym(h, "ncclAllGather");
        a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
        if (!a.get_unique_id || !a.comm_init_rank || !a.all_reduce || !a.all_gather) a.why = "libnccl symbols missing";
        return a;
    }();
    if (!api.why.empty()) throw cuda_error("NCCL: " + api.why);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw cuda_error(std::string("NCCL ") + what + ": " + (nccl().error_string ? nccl().error_string(r) : "error"));
}

}  // namespace

// ================================================================== comm
enum CommKind { COMM_LOCAL = 0, COMM_NCCL = 1, COMM_HOST = 2 };

struct vsr_comm {
    vsr_ctx* ctx = nullptr;
    int kind = COMM_LOCAL;
    int P = 1;
    int rank = 0;  // this process's rank (COMM_LOCAL: all ranks are local)
    ncclComm_t nc = nullptr;
    vsr_host_exchange ops{};
    void* user = nullptr;
    DevBuf<int> tick;
    std::vector<int> local_ranks() const {
        std::vector<int> r;
        if (kind == COMM_LOCAL)
            for (int p = 0; p < P; ++p) r.push_back(p);
        else
            r.push_back(rank);
        return r;
    }
    cudaStream_t stream() const { return vsr_capi::stream_of(ctx); }

    // stream-ordered barrier: every rank's work queued before it is complete
    // (and its peer stores visible) before any rank's work queued after it runs
    void barrier() {
        if (kind == COMM_LOCAL || P == 1) return;  // one stream: stream order is the barrier
        if (kind == COMM_NCCL) {
            nccl_check(nccl().all_reduce(tick.p, tick.p, 1, ncclInt, ncclSum, nc, stream()), "barrier");
            return;
        }
        VSR_CUDA(cudaStreamSynchronize(stream()));
        if (ops.barrier(user) != 0) throw cuda_error("vsr_comm: host barrier callback failed");
    }

    // all-gather of `bytes` host bytes per rank into out (P * bytes, rank order)
    void all_gather_host(const void* in, void* out, size_t bytes) {
        if (P == 1 || kind == COMM_LOCAL) {
            std::memcpy(out, in, bytes);
            return;
        }
        if (kind == COMM_HOST) {
            if (ops.all_gather(user, in, out, bytes) != 0) throw cuda_error("vsr_comm: host all_gather failed");
            return;
        }
        DevBuf<char> din(bytes), dout(bytes * P);
        cudaStream_t st = stream();
        VSR_CUDA(cudaMemcpyAsync(din.p, in, bytes, cudaMemcpyHostToDevice, st));
        nccl_check(nccl().all_gather(din.p, dout.p, bytes, ncclChar, nc, st), "all_gather");
        VSR_CUDA(cudaMemcpyAsync(out, dout.p, bytes * P, cudaMemcpyDeviceToHost, st));
        VSR_CUDA(cudaStreamSynchronize(st));
    }
};

namespace {

// Peer view of one buffer kind across ranks: ptr[q] is rank q's buffer as
// this process sees it (IPC-mapped for remote processes, plain for local ones).
struct PeerSet {
    std::vector<void*> ptr;
    std::vector<void*> opened;  // IPC mappings to close
    ~PeerSet() {
        for (void* p : opened) cudaIpcCloseMemHandle(p);
    }
};

// Exchanges `mine` (one pointer per local rank) into a P-entry peer table.
void share(vsr_comm* c, const std::vector<void*>& mine, PeerSet& out) {
    out.ptr.assign(c->P, nullptr);
    if (c->kind == COMM_LOCAL) {
        for (int p = 0; p < c->P; ++p) out.ptr[p] = mine[p];
        return;
    }
    out.ptr[c->rank] = mine[0];
    if (c->P == 1) return;
    cudaIpcMemHandle_t h{};
    VSR_CUDA(cudaIpcGetMemHandle(&h, mine[0]));
    std::vector<cudaIpcMemHandle_t> all(c->P);
    c->all_gather_host(&h, all.data(), sizeof(h));
    for (int q = 0; q < c->P; ++q) {
        if (q == c->rank) continue;
        void* p = nullptr;
        VSR_CUDA(cudaIpcOpenMemHandle(&p, all[q], cudaIpcMemLazyEnablePeerAccess));
        out.ptr[q] = p;
        out.opened.push_back(p);
    }
}

// ------------------------------------------------------------------ plan
// Plane ownership of the half spectrum (see the file comment).
struct SlabPlan {
    long long m = 0, n = 0, s = 0, nP = 0;
    int P = 1;
    FoldGeom G{};
    int half = 0;                    // s / 2 + 1 planes
    std::vector<int> owner;          // [half]: rank owning plane f3
    std::vector<int> wlocal;         // [half]: local plane index on its owner
    std::vector<std::vector<int>> planes;   // per rank: owned half planes (ascending)
    std::vector<std::vector<int>> classes;  // per rank: owned LR classes g3
    std::vector<std::vector<int>> lam_planes;  // per rank: full-spectrum planes f3 of its classes (ascending)
};

SlabPlan make_plan(const Spec& sp, int P) {
    SlabPlan pl;
    pl.m = (long long)sp.hr.m, pl.n = (long long)sp.hr.n, pl.s = (long long)sp.hr.s, pl.P = P;
    pl.G = make_geom(sp.hr, sp.rates);
    if (P < 1) throw std::invalid_argument("slab: rank count must be >= 1");
    if (pl.n % P) throw shape_error("slab: P=" + std::to_string(P) + " must divide axis 2 (" + std::to_string(pl.n) + ")");
    pl.nP = pl.n / P;
    if (pl.m % 2) throw shape_error("slab: axis 1 must be even");
    if (!fft_engine().half3_ok(Dims{(size_t)pl.m, (size_t)pl.nP, (size_t)pl.s}))
        throw shape_error("slab: axis 3 must be a power of two in [8, 1024] and m * n/P a multiple of 16");
    if (!fused_axis1_ok(pl.G)) throw shape_error("slab: no fused axis-1 fold for this geometry");
    const long long sl = pl.G.sl;
    pl.half = (int)(pl.s / 2 + 1);
    // conjugate class pairs {g, sl - g}, g = 0..sl/2, with their half-plane counts
    std::vector<std::vector<int>> pairs;
    std::vector<int> cnt;
    for (long long g = 0; g <= sl / 2; ++g) {
        std::vector<int> cls{(int)g};
        if (g != 0 && 2 * g != sl) cls.push_back((int)(sl - g));
        int c = 0;
        for (int f = 0; f < pl.half; ++f)
            for (int k : cls) c += (f % sl == k);
        pairs.push_back(cls);
        cnt.push_back(c);
    }
    if ((int)pairs.size() < P) throw shape_error("slab: P=" + std::to_string(P) + " exceeds the " +
                                                 std::to_string(pairs.size()) + " conjugate LR plane classes");
    // contiguous runs of pairs, balanced by half-plane count
    const int total = pl.half;
    pl.classes.assign(P, {});
    pl.planes.assign(P, {});
    pl.lam_planes.assign(P, {});
    // contiguous runs of pairs, balanced by half-plane count, at least one pair per rank
    std::vector<int> pair_rank(pairs.size()), npairs(P, 0);
    {
        int r = 0;
        long long acc = 0;
        const int np = (int)pairs.size();
        for (int i = 0; i < np; ++i) {
            const int ranks_after = P - 1 - r;
            if (r < P - 1 && npairs[r] > 0 && (acc * P >= (long long)(r + 1) * total || np - i <= ranks_after)) ++r;
            pair_rank[i] = r;
            ++npairs[r];
            acc += cnt[i];
        }
    }
    for (size_t i = 0; i < pairs.size(); ++i)
        for (int k : pairs[i]) pl.classes[pair_rank[i]].push_back(k);
    pl.owner.assign(pl.half, -1);
    pl.wlocal.assign(pl.half, -1);
    std::vector<int> cls_rank(sl, -1);
    for (int p = 0; p < P; ++p)
        for (int k : pl.classes[p]) cls_rank[k] = p;
    for (int f = 0; f < pl.half; ++f) {
        const int p = cls_rank[f % sl];
        pl.owner[f] = p;
        pl.wlocal[f] = (int)pl.planes[p].size();
        pl.planes[p].push_back(f);
    }
    for (long long f = 0; f < pl.s; ++f) pl.lam_planes[cls_rank[f % sl]].push_back((int)f);
    for (int p = 0; p < P; ++p)
        if (pl.planes[p].empty()) throw shape_error("slab: rank " + std::to_string(p) + " owns no spectral plane");
    return pl;
}

// ------------------------------------------------------------------ kernels
// x[i, j, k] of this rank's y-slab from y (nn_upsample, operators.cpp:155-164)
__global__ void slab_nn_upsample_kernel(long long m, long long nP, long long N, long long j0, int dr, int dc, int ds,
                                        long long ml, long long nl, const double* __restrict__ y,
                                        double* __restrict__ x) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= N) return;
    const long long i = p % m, j = j0 + (p / m) % nP, k = p / (m * nP);
    x[p] = y[(i / dr) + ml * ((j / dc) + nl * (k / ds))];
}

// fixed-order sums of this rank's per-block partials into hist[5 * it]:
// (fit, ||Lx - u||^2, sum ||Lx||, ||x - xprev||^2, ||xprev||^2)
__global__ void __launch_bounds__(1024)
    slab_scalars_kernel(int it, const double* __restrict__ fitp, long long nfit, const double* __restrict__ stp,
                        long long nst, double* __restrict__ hist) {
    __shared__ double red[32 * 4];
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (long long i = threadIdx.x; i < nfit; i += blockDim.x) v[0] += fitp[i];
    block_reduce_sum<4>(v, red);
    __syncthreads();
    const double fit = v[0];
    double w[4] = {0.0, 0.0, 0.0, 0.0};
    for (long long i = threadIdx.x; i < nst; i += blockDim.x)
        for (int q = 0; q < 4; ++q) w[q] += stp[4 * i + q];
    block_reduce_sum<4>(w, red);
    if (threadIdx.x == 0) {
        double* h = hist + 5 * (long long)it;
        h[0] = nfit ? fit : 0.0;
        h[1] = w[0];
        h[2] = w[1];
        h[3] = w[2];
        h[4] = w[3];
    }
}

// ------------------------------------------------------------------ per-rank state
struct Rank {
    int p = 0;
    Dims loc, spec;                        // (m, n/P, s) and (m, n, planes)
    DevBuf<double> x, xprev, theta, dualA, dualB;
    DevBuf<double2> W, W2, Yl, lam;        // lam: dense Lambda on lam planes (empty when separable)
    DevBuf<double2> sep;                   // a (m) | b (n) | c (s) when separable
    DevBuf<double> gw, tnr, tnc, tns;
    DevBuf<int> wplane, lplane, owner;
    DevBuf<long long> off;
    DevBuf<int2> tiles;
    int ntiles = 0;
    DevBuf<double2*> peerW, peerW2;
    DevBuf<double> fitp, stp, resp, hist;
    DevBuf<unsigned long long> bad;
    size_t st_blocks = 0, res_blocks = 0;
    const double* nb_x[2] = {nullptr, nullptr};  // lower / upper neighbour x
    const double* nb_dA = nullptr;               // lower neighbour dualA / dualB
    const double* nb_dB = nullptr;
};

struct SlabCommon {
    vsr_comm* comm = nullptr;
    Spec sp{};
    SlabPlan plan;
    std::vector<Rank> ranks;
    PeerSet pW, pW2, pX, pDA, pDB;
    bool separable = false;

    cudaStream_t st() const { return comm->stream(); }

    template <class F>
    void each(F&& f) {
        for (auto& r : ranks) f(r);
    }

    // per-rank tables of the plan; buffers of the spectral side
    void setup_rank(Rank& r, int p, bool tv_state) {
        const SlabPlan& pl = plan;
        cudaStream_t s = st();
        r.p = p;
        r.loc = Dims{(size_t)pl.m, (size_t)pl.nP, (size_t)pl.s};
        r.spec = Dims{(size_t)pl.m, (size_t)pl.n, pl.planes[p].size()};
        const size_t Nloc = r.loc.count(), Nspec = r.spec.count();
        r.x.alloc(Nloc);
        r.W.alloc(Nspec);
        r.W2.alloc(Nspec);
        if (tv_state) {
            r.theta.alloc(Nloc);
            r.dualA.alloc(3 * Nloc);
            r.dualB.alloc(3 * Nloc);
        }
        std::vector<int> wp(pl.half, -1), lp(pl.s, -1);
        for (size_t i = 0; i < pl.planes[p].size(); ++i) wp[pl.planes[p][i]] = (int)i;
        for (size_t i = 0; i < pl.lam_planes[p].size(); ++i) lp[pl.lam_planes[p][i]] = (int)i;
        std::vector<long long> off(pl.half);
        for (int f = 0; f < pl.half; ++f) off[f] = (long long)pl.wlocal[f] * pl.m * pl.n + (long long)p * pl.nP * pl.m;
        r.wplane.alloc(pl.half);
        r.lplane.alloc(pl.s);
        r.owner.alloc(pl.half);
        r.off.alloc(pl.half);
        VSR_CUDA(cudaMemcpyAsync(r.wplane.p, wp.data(), r.wplane.bytes(), cudaMemcpyHostToDevice, s));
        VSR_CUDA(cudaMemcpyAsync(r.lplane.p, lp.data(), r.lplane.bytes(), cudaMemcpyHostToDevice, s));
        VSR_CUDA(cudaMemcpyAsync(r.owner.p, pl.owner.data(), r.owner.bytes(), cudaMemcpyHostToDevice, s));
        VSR_CUDA(cudaMemcpyAsync(r.off.p, off.data(), r.off.bytes(), cudaMemcpyHostToDevice, s));
        // tiles (g2 block, g3) of this rank's classes
        const int T = tv_sandwich1_tile_g2(pl.G);
        std::vector<int2> tl;
        for (int g3 : pl.classes[p])
            for (long long b2 = 0; b2 < pl.G.nl / T; ++b2) tl.push_back(make_int2((int)b2, g3));
        std::sort(tl.begin(), tl.end(), [](int2 a, int2 b) { return a.y != b.y ? a.y < b.y : a.x < b.x; });
        r.ntiles = (int)tl.size();
        r.tiles.alloc(tl.size());
        VSR_CUDA(cudaMemcpyAsync(r.tiles.p, tl.data(), r.tiles.bytes(), cudaMemcpyHostToDevice, s));
        r.fitp.alloc(std::max(r.ntiles, 1));
        r.st_blocks = stencil_geom(r.loc).blocks();
        r.stp.alloc(kStencilVals * r.st_blocks);
        r.res_blocks = fft_engine().half3_blocks(r.loc);
        r.resp.alloc(2 * std::max<size_t>(r.res_blocks, 1));
        r.bad.alloc(1);
        VSR_CUDA(cudaMemsetAsync(r.bad.p, 0xff, sizeof(unsigned long long), s));
        VSR_CUDA(cudaStreamSynchronize(s));  // host tables above are stack-owned
    }

    void share_buffers(bool tv_state) {
        auto collect = [&](auto get) {
            std::vector<void*> v;
            for (auto& r : ranks) v.push_back((void*)get(r));
            return v;
        };
        share(comm, collect([](Rank& r) { return r.W.p; }), pW);
        share(comm, collect([](Rank& r) { return r.W2.p; }), pW2);
        share(comm, collect([](Rank& r) { return r.x.p; }), pX);
        if (tv_state) {
            share(comm, collect([](Rank& r) { return r.dualA.p; }), pDA);
            share(comm, collect([](Rank& r) { return r.dualB.p; }), pDB);
        }
        const int P = plan.P;
        for (auto& r : ranks) {
            std::vector<double2*> w(P), w2(P);
            for (int q = 0; q < P; ++q) w[q] = (double2*)pW.ptr[q], w2[q] = (double2*)pW2.ptr[q];
            r.peerW.alloc(P);
            r.peerW2.alloc(P);
            VSR_CUDA(cudaMemcpyAsync(r.peerW.p, w.data(), r.peerW.bytes(), cudaMemcpyHostToDevice, st()));
            VSR_CUDA(cudaMemcpyAsync(r.peerW2.p, w2.data(), r.peerW2.bytes(), cudaMemcpyHostToDevice, st()));
            VSR_CUDA(cudaStreamSynchronize(st()));
            const int lo = (r.p + P - 1) % P, hi = (r.p + 1) % P;
            r.nb_x[0] = (const double*)pX.ptr[lo];
            r.nb_x[1] = (const double*)pX.ptr[hi];
            if (tv_state) {
                r.nb_dA = (const double*)pDA.ptr[lo];
                r.nb_dB = (const double*)pDB.ptr[lo];
            }
        }
    }

    // Lambda (unnormalised DFT of the full PSF, or the given full spectrum) ->
    // separable 1-D tables or this rank's dense planes; Gw on the LR grid.
    void setup_lambda(const double2* lam_full_dev, const GammaTables& tabs_proto, bool want_gw) {
        const Dims hr = sp.hr;
        cudaStream_t s = st();
        for (auto& r : ranks) {
            r.sep.alloc(hr.m + hr.n + hr.s);
            separable = detect_separable(hr, lam_full_dev, r.sep.p, r.sep.p + hr.m, r.sep.p + hr.m + hr.n, 1e-13, s);
            if (!separable) {
                r.sep.release();
                const auto& lp = plan.lam_planes[r.p];
                r.lam.alloc((size_t)plan.m * plan.n * lp.size());
                for (size_t i = 0; i < lp.size(); ++i)
                    VSR_CUDA(cudaMemcpyAsync(r.lam.p + i * plan.m * plan.n, lam_full_dev + (size_t)lp[i] * plan.m * plan.n,
                                             (size_t)plan.m * plan.n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
            }
            if (want_gw) {
                r.gw.alloc(sp.lr.count());
                SepTables sept = sep_of(r);
                GammaTables t = tabs_proto;
                t.nr = r.tnr.p, t.nc = r.tnc.p, t.ns = r.tns.p;
                launch_tv_gram(plan.G, lam_full_dev, sept, t, r.gw.p, s);
            }
        }
        VSR_CUDA(cudaStreamSynchronize(s));
    }

    SepTables sep_of(const Rank& r) const {
        if (!r.sep.p) return SepTables{};
        return SepTables{r.sep.p, r.sep.p + sp.hr.m, r.sep.p + sp.hr.m + sp.hr.n};
    }

    void upload_tables(Rank& r, const std::vector<double>& nr, const std::vector<double>& nc,
                       const std::vector<double>& ns) {
        r.tnr.alloc(nr.size());
        r.tnc.alloc(nc.size());
        r.tns.alloc(ns.size());
        VSR_CUDA(cudaMemcpyAsync(r.tnr.p, nr.data(), r.tnr.bytes(), cudaMemcpyHostToDevice, st()));
        VSR_CUDA(cudaMemcpyAsync(r.tnc.p, nc.data(), r.tnc.bytes(), cudaMemcpyHostToDevice, st()));
        VSR_CUDA(cudaMemcpyAsync(r.tns.p, ns.data(), r.tns.bytes(), cudaMemcpyHostToDevice, st()));
        VSR_CUDA(cudaStreamSynchronize(st()));
    }

    GammaTables tabs_of(const Rank& r, double tau, int fit_only = 0) const {
        GammaTables t{r.tnr.p, r.tnc.p, r.tns.p, tau, r.gw.p, 1};
        t.wplane = r.wplane.p, t.lplane = r.lam.p ? r.lplane.p : nullptr, t.tiles = r.tiles.p, t.ntiles = r.ntiles;
        t.fit_only = fit_only;
        return t;
    }

    RemotePlanes remote(const Rank& r, bool inverse) const {
        return RemotePlanes{inverse ? r.peerW2.p : r.peerW.p, r.owner.p, r.off.p};
    }

    // forward: real y-slab `in` -> owners' W (axis 3 r2c + peer stores), barrier,
    // axis-2 forward on every local W
    void forward_to_W(const std::function<const double*(Rank&)>& in) {
        each([&](Rank& r) { fft_engine().r2c_axis3_half_remote(r.loc, in(r), remote(r, false), st()); });
        comm->barrier();
        each([&](Rank& r) {
            fft_engine().axis_pass(r.spec, 1, false, r.W.p, IN_COMPLEX, r.W.p, OUT_COMPLEX, 1.0, nullptr, st());
        });
    }

    // inverse: axis-2 inverse on every local W2, barrier, c2r pulling the
    // owners' planes into the x slabs (scaled; residue partials, bad index), barrier
    void inverse_to_x(double scale) {
        each([&](Rank& r) {
            fft_engine().axis_pass(r.spec, 1, true, r.W2.p, IN_COMPLEX, r.W2.p, OUT_COMPLEX, 1.0, nullptr, st());
        });
        comm->barrier();
        each([&](Rank& r) {
            PassReduce red{r.resp.p, r.bad.p};
            fft_engine().c2r_axis3_half_remote(r.loc, remote(r, true), r.x.p, scale, &red, st());
        });
        comm->barrier();
    }

    // LR spectrum of the full y on every rank (unitary)
    void lr_spectrum(const double* y_dev_full, Rank& r) {
        fft_engine().forward3(sp.lr, y_dev_full, IN_REAL, r.Yl.p, 1.0 / std::sqrt((double)sp.lr.count()), st());
    }

    // first non-finite flat index over all ranks (global lexicographic order), ULLONG_MAX if none
    unsigned long long first_bad() {
        std::vector<unsigned long long> mine;
        for (auto& r : ranks) {
            unsigned long long b = 0;
            VSR_CUDA(cudaMemcpyAsync(&b, r.bad.p, sizeof(b), cudaMemcpyDeviceToHost, st()));
            VSR_CUDA(cudaStreamSynchronize(st()));
            if (b != ULLONG_MAX) {  // local (m, nP, s) flat -> global (m, n, s)
                const unsigned long long i = b % plan.m, j = (b / plan.m) % plan.nP, k = b / (plan.m * plan.nP);
                b = i + plan.m * ((unsigned long long)r.p * plan.nP + j) + plan.m * plan.n * k;
            }
            mine.push_back(b);
        }
        std::vector<unsigned long long> all(comm->kind == COMM_LOCAL ? mine.size() : comm->P);
        if (comm->kind == COMM_LOCAL)
            all = mine;
        else
            comm->all_gather_host(mine.data(), all.data(), sizeof(unsigned long long));
        unsigned long long best = ULLONG_MAX;
        for (auto b : all) best = std::min(best, b);
        return best;
    }

    void reset_bad() {
        each([&](Rank& r) { VSR_CUDA(cudaMemsetAsync(r.bad.p, 0xff, sizeof(unsigned long long), st())); });
    }

    // gathers `count` doubles per rank from hist (device) in rank order
    std::vector<double> gather_hist(size_t count) {
        std::vector<double> mine(count * ranks.size());
        for (size_t i = 0; i < ranks.size(); ++i)
            VSR_CUDA(cudaMemcpyAsync(mine.data() + i * count, ranks[i].hist.p, count * sizeof(double),
                                     cudaMemcpyDeviceToHost, st()));
        VSR_CUDA(cudaStreamSynchronize(st()));
        if (comm->kind == COMM_LOCAL) return mine;
        std::vector<double> all(count * comm->P);
        comm->all_gather_host(mine.data(), all.data(), count * sizeof(double));
        return all;
    }
};

}  // namespace

// ================================================================== ADMM-TV
struct vsr_slab_tv : SlabCommon {
    double lambda = 0, mu = 0, rel_tol = 0, tau = 0;
    size_t max_iters = 0, iters_done = 0;
    bool dual_in_a = true, stopped = false;
    double init_objective = 0.0;
    std::vector<double> objective, residual;
    std::chrono::steady_clock::time_point t0;
};

namespace {

void tv_iteration(vsr_slab_tv* h) {
    const double s = 1.0 / std::sqrt((double)h->sp.hr.count());
    const double thr = h->lambda / h->mu;
    const int it = (int)h->iters_done;
    // theta_hat -> owners (axis 3 r2c + peer stores), axis 2 forward
    h->forward_to_W([](Rank& r) { return (const double*)r.theta.p; });
    // x-update fold (solvers.cpp:219-233) between the axis-1 transforms -> W2
    h->each([&](Rank& r) {
        launch_tv_sandwich1(h->plan.G, r.Yl.p, r.lam.p, r.W.p, h->tabs_of(r, h->tau), h->mu, s, r.fitp.p, h->st(),
                            h->sep_of(r), r.W2.p);
    });
    if (h->rel_tol > 0.0)
        h->each([&](Rank& r) {
            VSR_CUDA(cudaMemcpyAsync(r.xprev.p, r.x.p, r.x.bytes(), cudaMemcpyDeviceToDevice, h->st()));
        });
    // W2 -> x slabs (axis 2 inverse, barrier, c2r pulling the owners' planes, barrier)
    h->inverse_to_x(s);
    // shrink / dual / residual (:379-393) and theta for the next iteration (:367-373),
    // halos read from the neighbours' slabs in place
    h->each([&](Rank& r) {
        const bool a = h->dual_in_a;
        const double* din = a ? r.dualA.p : r.dualB.p;
        double* dout = a ? r.dualB.p : r.dualA.p;
        launch_tv_stencil_yslab(r.loc, false, r.x.p, din, dout, r.theta.p, thr,
                                h->rel_tol > 0.0 ? r.xprev.p : nullptr, r.stp.p, r.nb_x[0], r.nb_x[1],
                                a ? r.nb_dA : r.nb_dB, h->st());
        slab_scalars_kernel<<<1, 1024, 0, h->st()>>>(it, r.fitp.p, r.ntiles, r.stp.p, (long long)r.st_blocks,
                                                     r.hist.p);
        VSR_LAUNCH_CHECK();
    });
    h->dual_in_a = !h->dual_in_a;
    vsr_capi::add_fft_counts(1, 1);
    ++h->iters_done;
}

// objective / residual / rel change of iterations [from, to) summed over ranks in rank order
void tv_collect(vsr_slab_tv* h, size_t from, size_t to, double* last_rel) {
    const std::vector<double> all = h->gather_hist(5 * to);
    const size_t per = 5 * to, P = all.size() / per;
    for (size_t it = from; it < to; ++it) {
        double f = 0, r2 = 0, tv = 0, dx = 0, xp = 0;
        for (size_t p = 0; p < P; ++p) {
            const double* q = all.data() + p * per + 5 * it;
            f += q[0], r2 += q[1], tv += q[2], dx += q[3], xp += q[4];
        }
        h->objective.push_back(0.5 * f + h->lambda * tv);  // solvers.cpp:395-401
        h->residual.push_back(std::sqrt(r2));
        if (last_rel) *last_rel = std::sqrt(dx) / std::max(std::sqrt(xp), 1e-300);  // rel_change (:24-32)
    }
}

}  // namespace

extern "C" {

// unitary-scaled forward 3D FFT of device data (bench / tests: the engine alone)
int vsr_fft3_d(vsr_ctx* ctx, const size_t dims[3], const double* in, int in_real, double* out_c, double scale) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        const Dims d{dims[0], dims[1], dims[2]};
        if (d.count() == 0) throw shape_error("fft3: empty volume");
        fft_engine().forward3(d, in, in_real ? IN_REAL : IN_COMPLEX, reinterpret_cast<double2*>(out_c), scale,
                              vsr_capi::stream_of(ctx));
    });
}

int vsr_comm_local(vsr_ctx* ctx, int nranks, vsr_comm** out) {
    return vsr_capi::guard_call([&] {
        if (!ctx || !out) throw std::invalid_argument("vsr_comm_local: null argument");
        if (nranks < 1) throw std::invalid_argument("vsr_comm_local: nranks must be >= 1");
        DevGuard dg(vsr_capi::device_of(ctx));
        auto* c = new vsr_comm();
        c->ctx = ctx, c->kind = COMM_LOCAL, c->P = nranks, c->rank = 0;
        *out = c;
    });
}

int vsr_nccl_unique_id(unsigned char out[128]) {
    return vsr_capi::guard_call([&] {
        ncclUniqueId id;
        nccl_check(nccl().get_unique_id(&id), "get_unique_id");
        static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(out, &id, sizeof(id));
    });
}

int vsr_comm_nccl(vsr_ctx* ctx, int nranks, int rank, const unsigned char id[128], vsr_comm** out) {
    return vsr_capi::guard_call([&] {
        if (!ctx || !out || !id) throw std::invalid_argument("vsr_comm_nccl: null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("vsr_comm_nccl: bad rank");
        DevGuard dg(vsr_capi::device_of(ctx));
        auto* c = new vsr_comm();
        c->ctx = ctx, c->kind = COMM_NCCL, c->P = nranks, c->rank = rank;
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        try {
            nccl_check(nccl().comm_init_rank(&c->nc, nranks, uid, rank), "comm_init_rank");
            c->tick.alloc(1);
            VSR_CUDA(cudaMemset(c->tick.p, 0, sizeof(int)));
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int vsr_comm_host(vsr_ctx* ctx, int nranks, int rank, const vsr_host_exchange* ops, void* user, vsr_comm** out) {
    return vsr_capi::guard_call([&] {
        if (!ctx || !out || !ops || !ops->barrier || !ops->all_gather)
            throw std::invalid_argument("vsr_comm_host: null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("vsr_comm_host: bad rank");
        auto* c = new vsr_comm();
        c->ctx = ctx, c->kind = COMM_HOST, c->P = nranks, c->rank = rank, c->ops = *ops, c->user = user;
        *out = c;
    });
}

int vsr_comm_destroy(vsr_comm* c) {
    return vsr_capi::guard_call([&] {
        if (!c) return;
        DevGuard dg(vsr_capi::device_of(c->ctx));
        if (c->nc && nccl().comm_destroy) nccl().comm_destroy(c->nc);
        delete c;
    });
}

int vsr_comm_info(vsr_comm* c, int* nranks, int* rank, int* local_ranks) {
    return vsr_capi::guard_call([&] {
        if (!c) throw std::invalid_argument("vsr_comm_info: null comm");
        if (nranks) *nranks = c->P;
        if (rank) *rank = c->kind == COMM_LOCAL ? -1 : c->rank;
        if (local_ranks) *local_ranks = (int)c->local_ranks().size();
    });
}

int vsr_slab_plan(const size_t hr_dims[3], const size_t rates[3], int nranks, int rank, int* owner_half,
                  int* nplanes) {
    return vsr_capi::guard_call([&] {
        const Spec sp = make_spec(hr_dims, rates);
        const SlabPlan pl = make_plan(sp, nranks);
        if (rank < 0 || rank >= nranks) throw std::invalid_argument("vsr_slab_plan: bad rank");
        if (owner_half)
            for (int f = 0; f < pl.half; ++f) owner_half[f] = pl.owner[f];
        if (nplanes) *nplanes = (int)pl.planes[rank].size();
    });
}

int vsr_slab_tv_create(vsr_comm* comm, const size_t hr_dims[3], const size_t rates[3], const double* y_r,
                       const double* psf_r, const vsr_tv_config* cfg, const double* const* init_slabs,
                       vsr_slab_tv** out) {
    return vsr_capi::guard_call([&] {
        if (!comm || !out || !cfg || !y_r || !psf_r) throw std::invalid_argument("vsr_slab_tv_create: null argument");
        DevGuard dg(vsr_capi::device_of(comm->ctx));
        if (!(cfg->lambda > 0.0))
            throw std::invalid_argument("lambda must be positive, got " + std::to_string(cfg->lambda));
        if (!(cfg->mu > 0.0)) throw std::invalid_argument("mu must be positive, got " + std::to_string(cfg->mu));
        if (cfg->max_iters < 1) throw std::invalid_argument("admm_tv: max_iters must be >= 1");
        if (cfg->precision != VSR_PRECISION_F64)
            throw std::invalid_argument("admm_tv: the slab-sharded path runs in fp64 only");
        auto* h = new vsr_slab_tv();
        try {
            h->t0 = std::chrono::steady_clock::now();
            h->comm = comm;
            h->sp = make_spec(hr_dims, rates);
            h->plan = make_plan(h->sp, comm->P);
            h->lambda = cfg->lambda, h->mu = cfg->mu, h->rel_tol = cfg->rel_tol, h->max_iters = cfg->max_iters;
            h->tau = cfg->has_tau ? cfg->tau : 1e-8 * cfg->mu;  // solvers.cpp:332
            validate_tau(h->tau);
            const Dims hr = h->sp.hr, lr = h->sp.lr;
            cudaStream_t st = h->st();
            const auto lr_ranks = comm->local_ranks();
            h->ranks.resize(lr_ranks.size());
            const auto nr = diff_norm_table(hr.m), nc = diff_norm_table(hr.n), ns = diff_norm_table(hr.s);
            for (size_t i = 0; i < lr_ranks.size(); ++i) {
                Rank& r = h->ranks[i];
                h->setup_rank(r, lr_ranks[i], true);
                h->upload_tables(r, nr, nc, ns);
                if (h->rel_tol > 0.0) r.xprev.alloc(r.loc.count());
                r.hist.alloc(5 * h->max_iters + 5);
                r.Yl.alloc(lr.count());
            }
            h->share_buffers(true);
            // precompute (solvers.cpp:336-344): Lambda = DFT(psf) on every rank, then
            // its separable factors or this rank's planes; Gw; the LR spectrum of y
            {
                DevBuf<double> psf(hr.count()), y(lr.count());
                DevBuf<double2> lam(hr.count());
                VSR_CUDA(cudaMemcpyAsync(psf.p, psf_r, psf.bytes(), cudaMemcpyHostToDevice, st));
                VSR_CUDA(cudaMemcpyAsync(y.p, y_r, y.bytes(), cudaMemcpyHostToDevice, st));
                fft_engine().forward3(hr, psf.p, IN_REAL, lam.p, 1.0, st);
                GammaTables proto{nullptr, nullptr, nullptr, h->tau};
                h->setup_lambda(lam.p, proto, true);
                for (auto& r : h->ranks) h->lr_spectrum(y.p, r);
                vsr_capi::add_fft_counts(2, 0);
                // init (solvers.cpp:346-354)
                for (size_t i = 0; i < h->ranks.size(); ++i) {
                    Rank& r = h->ranks[i];
                    if (cfg->init == VSR_INIT_ZERO) {
                        VSR_CUDA(cudaMemsetAsync(r.x.p, 0, r.x.bytes(), st));
                    } else if (cfg->init == VSR_INIT_UPSAMPLED) {
                        const long long N = (long long)r.loc.count();
                        slab_nn_upsample_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(
                            (long long)hr.m, h->plan.nP, N, (long long)r.p * h->plan.nP, h->sp.rates[0],
                            h->sp.rates[1], h->sp.rates[2], (long long)lr.m, (long long)lr.n, y.p, r.x.p);
                        VSR_LAUNCH_CHECK();
                    } else if (cfg->init == VSR_INIT_PROVIDED) {
                        if (!init_slabs || !init_slabs[i]) throw shape_error("admm_tv: init volume: dims mismatch");
                        VSR_CUDA(cudaMemcpyAsync(r.x.p, init_slabs[i], r.x.bytes(), cudaMemcpyHostToDevice, st));
                    } else {
                        throw std::invalid_argument("admm_tv: unknown init mode");
                    }
                }
                VSR_CUDA(cudaStreamSynchronize(st));
            }
            comm->barrier();  // every x0 slab in place before the neighbours' halo reads
            // u0 = L x0, dual0 = 0 (:356-358) -> theta of iteration 1; TV(x0)
            const double thr = h->lambda / h->mu;
            h->each([&](Rank& r) {
                launch_tv_stencil_yslab(r.loc, true, r.x.p, nullptr, r.dualA.p, r.theta.p, thr, nullptr, r.stp.p,
                                        r.nb_x[0], r.nb_x[1], nullptr, st);
            });
            // initial objective (:361): data fit of fft3(x0) by LR Parseval
            h->forward_to_W([](Rank& r) { return (const double*)r.x.p; });
            const double s = 1.0 / std::sqrt((double)hr.count());
            h->each([&](Rank& r) {
                launch_tv_sandwich1(h->plan.G, r.Yl.p, r.lam.p, r.W.p, h->tabs_of(r, h->tau, 1), h->mu, s, r.fitp.p,
                                    st, h->sep_of(r), r.W2.p);
                slab_scalars_kernel<<<1, 1024, 0, st>>>((int)h->max_iters, r.fitp.p, r.ntiles, r.stp.p,
                                                        (long long)r.st_blocks, r.hist.p);
                VSR_LAUNCH_CHECK();
            });
            vsr_capi::add_fft_counts(1, 0);
            comm->barrier();  // the next forward rewrites W
            const std::vector<double> all = h->gather_hist(5 * h->max_iters + 5);
            const size_t per = 5 * h->max_iters + 5;
            double f = 0, tv = 0;
            for (size_t p = 0; p < all.size() / per; ++p) {
                f += all[p * per + 5 * h->max_iters];
                tv += all[p * per + 5 * h->max_iters + 2];
            }
            h->init_objective = 0.5 * f + h->lambda * tv;
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int vsr_slab_tv_iterate(vsr_slab_tv* h, size_t iters) {
    return vsr_capi::guard_call([&] {
        if (!h) throw std::invalid_argument("vsr_slab_tv_iterate: null handle");
        DevGuard dg(vsr_capi::device_of(h->comm->ctx));
        const size_t start = h->iters_done;
        for (size_t k = 0; k < iters && !h->stopped && h->iters_done < h->max_iters; ++k) {
            tv_iteration(h);
            if (h->rel_tol > 0.0) {  // stop rule (solvers.cpp:405): scalars every iteration
                double rel = 0.0;
                tv_collect(h, h->iters_done - 1, h->iters_done, &rel);
                if (rel < h->rel_tol) h->stopped = true;
            }
        }
        if (h->rel_tol <= 0.0 && h->iters_done > start) tv_collect(h, start, h->iters_done, nullptr);
    });
}

int vsr_slab_tv_local_ranks(vsr_slab_tv* h, int* count) {
    return vsr_capi::guard_call([&] { *count = (int)h->ranks.size(); });
}

// x slabs (one per local rank, (m, n/P, s) each) on the device
int vsr_slab_tv_x_d(vsr_slab_tv* h, int local, const double** x_dev) {
    return vsr_capi::guard_call([&] {
        if (!h || local < 0 || local >= (int)h->ranks.size()) throw std::out_of_range("vsr_slab_tv_x_d: local rank");
        *x_dev = h->ranks[local].x.p;
    });
}

int vsr_slab_tv_finish(vsr_slab_tv* h, double* const* x_slabs, vsr_report* rep) {
    return vsr_capi::guard_call([&] {
        if (!h) throw std::invalid_argument("vsr_slab_tv_finish: null handle");
        DevGuard dg(vsr_capi::device_of(h->comm->ctx));
        VSR_CUDA(cudaStreamSynchronize(h->st()));
        const unsigned long long bad = h->first_bad();  // require_finite(x, "admm_tv") (:408)
        if (bad != ULLONG_MAX) {
            h->reset_bad();
            throw numeric_error("admm_tv: non-finite value at flat index " + std::to_string(bad));
        }
        if (x_slabs)
            for (size_t i = 0; i < h->ranks.size(); ++i)
                if (x_slabs[i])
                    VSR_CUDA(cudaMemcpyAsync(x_slabs[i], h->ranks[i].x.p, h->ranks[i].x.bytes(), cudaMemcpyDeviceToHost,
                                             h->st()));
        VSR_CUDA(cudaStreamSynchronize(h->st()));
        if (rep) {
            rep->iterations = h->iters_done;
            rep->initial_objective = h->init_objective;
            rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - h->t0).count();
            for (size_t i = 0; i < h->objective.size(); ++i) {
                if (rep->objective) rep->objective[i] = h->objective[i];
                if (rep->primal_residual) rep->primal_residual[i] = h->residual[i];
            }
        }
    });
}

int vsr_slab_tv_destroy(vsr_slab_tv* h) {
    return vsr_capi::guard_call([&] {
        if (!h) return;
        DevGuard dg(vsr_capi::device_of(h->comm->ctx));
        cudaStreamSynchronize(h->st());
        // every rank is done with the peers' buffers before anyone frees its own
        try {
            h->comm->barrier();
        } catch (...) {
        }
        cudaStreamSynchronize(h->st());
        delete h;
    });
}

int vsr_slab_admm_tv(vsr_comm* comm, const size_t hr_dims[3], const size_t rates[3], const double* y_r,
                     const double* psf_r, const vsr_tv_config* cfg, const double* const* init_slabs,
                     double* const* x_slabs, vsr_report* rep) {
    vsr_slab_tv* h = nullptr;
    int rc = vsr_slab_tv_create(comm, hr_dims, rates, y_r, psf_r, cfg, init_slabs, &h);
    if (rc != VSR_OK) return rc;
    rc = vsr_slab_tv_iterate(h, cfg->max_iters);
    if (rc == VSR_OK) rc = vsr_slab_tv_finish(h, x_slabs, rep);
    vsr_slab_tv_destroy(h);
    return rc;
}

}  // extern "C"

// ================================================================== Tikhonov
// TikhonovOperator (solvers.cpp:36-67) on the same decomposition.  The closed
// form is the TV sandwich with Gamma = 1 (zero difference tables, tau = 1),
// mu = 2 reg and theta_hat = fft3(xbar): k = conj(L) F D^H y + 2 reg X̄,
// w = fold(L k) / (gram + 2 reg d), x̂ = (k - conj(L) w) / (2 reg).  X̄ is
// transformed into W once; each solve is the LR spectrum of y, the sandwich
// into W2 and the distributed inverse.
struct vsr_slab_tikhonov : SlabCommon {
    double reg = 0;
    DevBuf<double> ydev;
};

extern "C" {

int vsr_slab_tikhonov_create(vsr_comm* comm, const size_t hr_dims[3], const size_t rates[3], const double* lambda_c,
                             double reg, const double* const* xbar_slabs, vsr_slab_tikhonov** out) {
    return vsr_capi::guard_call([&] {
        if (!comm || !out || !lambda_c || !xbar_slabs) throw std::invalid_argument("vsr_slab_tikhonov_create: null argument");
        DevGuard dg(vsr_capi::device_of(comm->ctx));
        require_positive(reg, "lambda");  // solvers.cpp:39
        auto* h = new vsr_slab_tikhonov();
        try {
            h->comm = comm;
            h->sp = make_spec(hr_dims, rates);
            h->plan = make_plan(h->sp, comm->P);
            h->reg = reg;
            const Dims hr = h->sp.hr, lr = h->sp.lr;
            cudaStream_t st = h->st();
            const auto lr_ranks = comm->local_ranks();
            h->ranks.resize(lr_ranks.size());
            const std::vector<double> zr(hr.m, 0.0), zc(hr.n, 0.0), zs(hr.s, 0.0);
            for (size_t i = 0; i < lr_ranks.size(); ++i) {
                Rank& r = h->ranks[i];
                h->setup_rank(r, lr_ranks[i], false);
                h->upload_tables(r, zr, zc, zs);  // Gamma = 1 / (0 + 1)
                r.Yl.alloc(lr.count());
            }
            h->ydev.alloc(lr.count());
            h->share_buffers(false);
            {
                DevBuf<double2> lam(hr.count());
                VSR_CUDA(cudaMemcpyAsync(lam.p, lambda_c, lam.bytes(), cudaMemcpyHostToDevice, st));
                GammaTables proto{nullptr, nullptr, nullptr, 1.0};
                h->setup_lambda(lam.p, proto, true);  // Gw = gram_diag (spectral.cpp:125-131)
            }
            // xbar_hat_ = fft3(xbar) (:45), kept in W on its owners (axes 3, 2; the
            // sandwich applies axis 1 and the unitary scale)
            for (size_t i = 0; i < h->ranks.size(); ++i)
                VSR_CUDA(cudaMemcpyAsync(h->ranks[i].x.p, xbar_slabs[i], h->ranks[i].x.bytes(), cudaMemcpyHostToDevice,
                                         st));
            VSR_CUDA(cudaStreamSynchronize(st));
            h->forward_to_W([](Rank& r) { return (const double*)r.x.p; });
            vsr_capi::add_fft_counts(1, 0);
            h->comm->barrier();
            VSR_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

static void slab_tik_enqueue(vsr_slab_tikhonov* h, const double* y_dev) {
    const double s = 1.0 / std::sqrt((double)h->sp.hr.count());
    h->reset_bad();
    h->each([&](Rank& r) {
        h->lr_spectrum(y_dev, r);  // F D^H y in LR form (the one forward transform, :52)
        launch_tv_sandwich1(h->plan.G, r.Yl.p, r.lam.p, r.W.p, h->tabs_of(r, 1.0), 2.0 * h->reg, s, nullptr, h->st(),
                            h->sep_of(r), r.W2.p);
    });
    h->inverse_to_x(s);  // x = ifft3_real(x̂) (:64), real by construction
    vsr_capi::add_fft_counts(1, 1);
}

static void slab_tik_check(vsr_slab_tikhonov* h) {
    const unsigned long long bad = h->first_bad();
    if (bad != ULLONG_MAX) {
        h->reset_bad();
        throw numeric_error("tikhonov_fast: non-finite value at flat index " + std::to_string(bad));
    }
}

int vsr_slab_tikhonov_solve(vsr_slab_tikhonov* h, const double* y_r, double* const* x_slabs) {
    return vsr_capi::guard_call([&] {
        if (!h || !y_r) throw std::invalid_argument("vsr_slab_tikhonov_solve: null argument");
        DevGuard dg(vsr_capi::device_of(h->comm->ctx));
        VSR_CUDA(cudaMemcpyAsync(h->ydev.p, y_r, h->ydev.bytes(), cudaMemcpyHostToDevice, h->st()));
        slab_tik_enqueue(h, h->ydev.p);
        slab_tik_check(h);  // require_finite (:65)
        if (x_slabs)
            for (size_t i = 0; i < h->ranks.size(); ++i)
                if (x_slabs[i])
                    VSR_CUDA(cudaMemcpyAsync(x_slabs[i], h->ranks[i].x.p, h->ranks[i].x.bytes(), cudaMemcpyDeviceToHost,
                                             h->st()));
        VSR_CUDA(cudaStreamSynchronize(h->st()));
    });
}

// device-resident solve: y (full LR, device) -> the rank's x slab stays on the
// device (vsr_slab_tikhonov_x_d); no host synchronisation
int vsr_slab_tikhonov_solve_d(vsr_slab_tikhonov* h, const double* y_dev) {
    return vsr_capi::guard_call([&] {
        if (!h || !y_dev) throw std::invalid_argument("vsr_slab_tikhonov_solve_d: null argument");
        DevGuard dg(vsr_capi::device_of(h->comm->ctx));
        slab_tik_enqueue(h, y_dev);
    });
}

int vsr_slab_tikhonov_check(vsr_slab_tikhonov* h) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(h->comm->ctx));
        slab_tik_check(h);
    });
}

int vsr_slab_tikhonov_x_d(vsr_slab_tikhonov* h, int local, const double** x_dev) {
    return vsr_capi::guard_call([&] {
        if (!h || local < 0 || local >= (int)h->ranks.size())
            throw std::out_of_range("vsr_slab_tikhonov_x_d: local rank");
        *x_dev = h->ranks[local].x.p;
    });
}

int vsr_slab_tikhonov_destroy(vsr_slab_tikhonov* h) {
    return vsr_capi::guard_call([&] {
        if (!h) return;
        DevGuard dg(vsr_capi::device_of(h->comm->ctx));
        cudaStreamSynchronize(h->st());
        try {
            h->comm->barrier();
        } catch (...) {
        }
        cudaStreamSynchronize(h->st());
        delete h;
    });
}

}  // extern "C"
