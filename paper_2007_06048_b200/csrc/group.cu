// group.cu -- multi-GPU z-slab execution of acoustic_iso_cd behind the C ABI
// (mm_cd_group_*), one process (rank) per GPU, halo planes over NCCL.
//
// ref: run_distributed_rank (dist.cpp:144-267) and exchange_halos
// (dist.cpp:92-115); legality of the cuts, validate_cuts (dist.cpp:119-132).
//
// B200 design:
//  * the global grid is cut along z, the slowest axis of the device layout,
//    so a rank's r owned edge planes and its r ghost planes are contiguous
//    blocks: NCCL sends / receives them in place, no packing kernels;
//  * legal cuts (nd + r <= cut <= n - nd - r) keep every CPML memory read
//    inside its rank, so only p is exchanged, as in the reference;
//  * one step (the "overlap" schedule):
//      CPML pass 1 (all planes) -> [edge stream] p_next on the r planes next
//      to each cut (+ the source when it sits there) -> [comm stream]
//      ncclSend/ncclRecv of those planes into the neighbours' p_next ghost
//      planes || [engine stream] the interior planes (interior kernel beside
//      the boundary kernel) -> join -> epilogue (source, free surface on
//      rank 0, receivers, the rank's finiteness check at its slab centre,
//      dist.cpp:222-224) -> rotate.
//    The exchanged planes become the neighbours' p_cur ghosts after the
//    rotation: what the reference's exchange_halos(p_cur) produces before the
//    next step, so the slabs are bit-identical to one engine on the whole
//    grid.
//  * NCCL is resolved at run time (dlopen of libnccl.so.2: the copy a host
//    runtime such as torch already loaded, else the system one), so the
//    single-GPU library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/minimod_b200.h"
#include "cd_engine.hpp"

namespace mmb {
namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = nullptr;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            api.why = std::string("libnccl.so.2 not found: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart &&
                 api.GroupEnd && api.Send && api.Recv && api.GetErrorString;
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    if (!api.ok) raise(ST_NCCL, "NCCL unavailable: " + api.why);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        raise(ST_NCCL, std::string("NCCL error in ") + what + ": " + nccl().GetErrorString(r));
}

}  // namespace
}  // namespace mmb

struct mm_cd_group {
    mm_cd_engine* e = nullptr;  // the rank's slab engine (owned)
    int rank = 0, world = 1;
    std::vector<int> cuts;      // z cuts of the global grid, world + 1 entries
    int gn[3] = {0, 0, 0};
    int z0 = 0, nz = 0;
    ncclComm_t comm = nullptr;
    cudaStream_t cs = nullptr;  // communication stream
    cudaStream_t es = nullptr;  // edge-plane stream
    cudaEvent_t ev_p1 = nullptr, ev_edges = nullptr, ev_comm = nullptr;
    bool lower = false, upper = false;  // neighbours below / above
    int edges[4] = {0, 0, 0, 0};        // plane ranges next to the cuts
    int nedge = 0;
    int ilo = 0, ihi = 0;               // interior plane range
    bool side = false;                  // this step's interior kernel runs on the side stream
    long long centre = 0;               // device offset of the slab centre (finiteness check)

    ~mm_cd_group() {
        if (e) {
            cudaSetDevice(e->device);
            cudaStreamSynchronize(e->stream);
        }
        if (cs) {
            cudaStreamSynchronize(cs);
            cudaStreamDestroy(cs);
        }
        if (es) {
            cudaStreamSynchronize(es);
            cudaStreamDestroy(es);
        }
        if (ev_p1) cudaEventDestroy(ev_p1);
        if (ev_edges) cudaEventDestroy(ev_edges);
        if (ev_comm) cudaEventDestroy(ev_comm);
        if (comm) mmb::nccl().CommDestroy(comm);
        if (e) mm_cd_destroy(e);
    }

    // src_global -> local offset if this rank owns it (else -1)
    long long local_src(const int* src) const {
        if (!src) return -1;
        for (int a = 0; a < 3; ++a)
            if (src[a] < 0 || src[a] >= gn[a])
                mmb::raise(mmb::ST_CONFIG, "source location outside grid interior");
        if (src[2] < z0 || src[2] >= z0 + nz) return -1;
        return e->lay.off(src[0], src[1], src[2] - z0);
    }
    bool in_edges(long long off) const {
        if (off < 0) return false;
        const int k = (int)(off / e->lay.plane) - e->lay.r;
        for (int i = 0; i < nedge; ++i)
            if (k >= edges[2 * i] && k < edges[2 * i + 1]) return true;
        return false;
    }

    // One step of the overlap schedule (see the file comment), in two phases
    // so an in-process test can interleave several ranks (step_local):
    //   phase 1: pass 1, the edge planes (edge stream), the halo transfer
    //            (communication stream: NCCL, or `local_peers` copies);
    //   phase 2: the interior planes, the join, the epilogue, the rotation.
    // amp_dev / step_dev: device wavelet + step counter (device loop) or null.
    struct StepArgs {
        float amp;
        long long so;
        const float* amp_dev;
        int* step_dev;
        const mmb::RecParams* rec;
    };
    mm_cd_group** local_peers = nullptr;  // in-process ranks (tests), else NCCL

    void phase1(const StepArgs& a) {
        using namespace mmb;
        mm_cd_engine& E = *e;
        const StepParams sp = E.params();
        const bool fst = E.mode != MM_MODE_STRICT && E.fast;
        E.flush_epilogue();  // a host-driven mm_cd_step on this engine before the group's
        // the interior planes need p_cur only: forked from the step's start,
        // beside pass 1 (the single-engine step's overlap)
        side = false;
        if (fst && ihi > ilo) E.fast->fork_point(E.stream);
        E.pass1();
        if (fst && ihi > ilo) side = E.fast->interior_side(sp, ilo, ihi);
        // the planes next to the cuts on their own stream, issued first (the
        // persistent interior kernels then fill the SMs they leave), so the
        // transfer waits for them only, not for the interior
        MM_CUDA(cudaEventRecord(ev_p1, E.stream));
        MM_CUDA(cudaStreamWaitEvent(es, ev_p1, 0));
        if (nedge) {
            if (fst)
                E.fast->update_ranges(sp, edges, nedge, es);
            else
                for (int i = 0; i < nedge; ++i) strict_update(sp, 0, edges[2 * i], edges[2 * i + 1], es);
        }
        if (in_edges(a.so)) launch_inject(sp.pn, sp.cv, a.so, a.amp, a.amp_dev, a.step_dev, es);
        // halo planes of p_next: owned edge planes -> the neighbours' ghosts
        MM_CUDA(cudaEventRecord(ev_edges, es));
        MM_CUDA(cudaStreamWaitEvent(cs, ev_edges, 0));
        const int r = E.lay.r;
        const size_t count = (size_t)r * E.lay.plane;
        float* pn = E.p[E.in].ptr;
        float* own_lo = pn + (long long)r * E.lay.plane;        // planes [0, r)
        float* own_hi = pn + (long long)nz * E.lay.plane;       // planes [nz - r, nz)
        if (local_peers) {
            // in place of NCCL: write my edge planes into the neighbours' ghosts
            if (lower) {
                mm_cd_engine& D = *local_peers[rank - 1]->e;
                float* dst = D.p[D.in].ptr + (long long)(local_peers[rank - 1]->nz + r) * D.lay.plane;
                MM_CUDA(cudaMemcpyAsync(dst, own_lo, count * 4, cudaMemcpyDeviceToDevice, cs));
            }
            if (upper) {
                mm_cd_engine& D = *local_peers[rank + 1]->e;
                MM_CUDA(cudaMemcpyAsync(D.p[D.in].ptr, own_hi, count * 4, cudaMemcpyDeviceToDevice,
                                        cs));
            }
        } else if (lower || upper) {
            const NcclApi& N = nccl();
            nccl_check(N.GroupStart(), "ncclGroupStart");
            if (lower) {
                nccl_check(N.Send(own_lo, count, ncclFloat, rank - 1, comm, cs), "ncclSend");
                nccl_check(N.Recv(pn, count, ncclFloat, rank - 1, comm, cs), "ncclRecv");
            }
            if (upper) {
                nccl_check(N.Send(own_hi, count, ncclFloat, rank + 1, comm, cs), "ncclSend");
                nccl_check(N.Recv(pn + (long long)(nz + r) * E.lay.plane, count, ncclFloat,
                                  rank + 1, comm, cs),
                           "ncclRecv");
            }
            nccl_check(N.GroupEnd(), "ncclGroupEnd");
        }
        MM_CUDA(cudaEventRecord(ev_comm, cs));
    }

    void phase2(const StepArgs& a) {
        using namespace mmb;
        mm_cd_engine& E = *e;
        const StepParams sp = E.params();
        const bool fst = E.mode != MM_MODE_STRICT && E.fast;
        // the interior planes' boundary kernel (the interior kernel is already
        // running on the side stream), concurrent with the transfer
        if (ihi > ilo) {
            if (fst)
                E.fast->finish_overlap(sp, ilo, ihi, E.stream, side);
            else
                E.update(0, ilo, ihi);
        }
        MM_CUDA(cudaStreamWaitEvent(E.stream, ev_edges, 0));
        MM_CUDA(cudaStreamWaitEvent(E.stream, ev_comm, 0));
        if (local_peers) {  // the neighbours' copies into my ghosts
            if (lower) MM_CUDA(cudaStreamWaitEvent(E.stream, local_peers[rank - 1]->ev_comm, 0));
            if (upper) MM_CUDA(cudaStreamWaitEvent(E.stream, local_peers[rank + 1]->ev_comm, 0));
        }
        Epilogue ep;
        std::memset(&ep, 0, sizeof ep);
        ep.p = sp.pn;
        ep.cv = sp.cv;
        ep.src_off = in_edges(a.so) ? -1LL : a.so;
        ep.amp = a.amp;
        ep.amp_dev = a.amp_dev;
        ep.step_dev = a.step_dev;
        ep.count = a.step_dev != nullptr;
        ep.fs = E.free_surface && E.goff[2] == 0;
        ep.lay = E.lay;
        if (a.rec) ep.rec = *a.rec;
        ep.check_off = a.rec && a.rec->bad_step ? centre : -1;
        ep.done = E.counters.ptr + 2;
        // a host-driven step's epilogue waits for the next call on the engine,
        // as in mm_cd_step: a following mm_cd_record samples inside it
        if (!a.amp_dev && !a.step_dev && !a.rec && tuning("defer_epilogue") != 0) {
            E.pending_ep = ep;
            E.ep_pending = true;
        } else {
            launch_epilogue(ep, E.stream);
        }
        E.rotate();
        ++E.steps;
    }

    void step(float amp, long long so, const float* amp_dev, int* step_dev,
              const mmb::RecParams* rec) {
        const StepArgs a{amp, so, amp_dev, step_dev, rec};
        phase1(a);
        phase2(a);
    }
};

using namespace mmb;

extern "C" {

int mm_nccl_get_unique_id(unsigned char id[128]) {
    MM_API_BEGIN
    need(id, "id");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof u);
    MM_API_END
}

int mm_zslab_validate_cuts(const int* cuts, int world, int nz, int ndamping_z, int radius) {
    MM_API_BEGIN
    need(cuts, "cuts");
    if (world < 1) raise(ST_CONFIG, "world size must be >= 1");
    if (cuts[0] != 0 || cuts[world] != nz) raise(ST_CONFIG, "cuts must start at 0 and end at nz");
    const int keep = ndamping_z + radius;
    for (int c = 1; c < world; ++c)  // dist.cpp:119-132
        if (cuts[c] < keep || cuts[c] > nz - keep)
            raise(ST_CONFIG, "rank boundary at index " + std::to_string(cuts[c]) +
                                 " cuts through the damping region (must be >= " +
                                 std::to_string(keep) + " points from either domain boundary)");
    for (int c = 0; c < world; ++c)
        if (cuts[c + 1] - cuts[c] < radius)
            raise(ST_CONFIG, "slab [" + std::to_string(cuts[c]) + ", " + std::to_string(cuts[c + 1]) +
                                 ") is thinner than the stencil radius");
    MM_API_END
}

int mm_cd_group_create(const mm_grid* global, const int* cuts, int world, int rank,
                       const unsigned char nccl_id[128], const float* vp_local,
                       const mm_engine_options* opts, float dt, double vmax, int device, int mode,
                       mm_cd_group** out) {
    MM_API_BEGIN
    need(global, "global grid");
    need(cuts, "cuts");
    need(out, "out");
    need(opts, "options");
    *out = nullptr;
    if (rank < 0 || rank >= world) raise(ST_INVAL, "rank out of range");
    int rc = mm_zslab_validate_cuts(cuts, world, global->n[2], opts->ndamping[2], global->radius);
    if (rc) return rc;
    auto g = std::make_unique<mm_cd_group>();
    g->rank = rank;
    g->world = world;
    g->cuts.assign(cuts, cuts + world + 1);
    for (int a = 0; a < 3; ++a) g->gn[a] = global->n[a];
    g->z0 = cuts[rank];
    g->nz = cuts[rank + 1] - cuts[rank];
    mm_grid lg = *global;
    lg.n[2] = g->nz;
    const int off[3] = {0, 0, g->z0};
    rc = mm_cd_create(&lg, off, global->n, vp_local, opts, dt, vmax, device, mode, &g->e);
    if (rc) return rc;
    MM_CUDA(cudaSetDevice(device));
    // the edge planes and the halo transfer gate the neighbours' next step:
    // their streams at the greatest priority, so their CTAs are dispatched
    // before the interior and boundary kernels of the same step
    int prio_lo = 0, prio_hi = 0;
    MM_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    MM_CUDA(cudaStreamCreateWithPriority(&g->cs, cudaStreamNonBlocking, prio_hi));
    MM_CUDA(cudaStreamCreateWithPriority(&g->es, cudaStreamNonBlocking, prio_hi));
    MM_CUDA(cudaEventCreateWithFlags(&g->ev_p1, cudaEventDisableTiming));
    MM_CUDA(cudaEventCreateWithFlags(&g->ev_edges, cudaEventDisableTiming));
    MM_CUDA(cudaEventCreateWithFlags(&g->ev_comm, cudaEventDisableTiming));
    g->lower = rank > 0;
    g->upper = rank + 1 < world;
    const int r = global->radius, nz = g->nz;
    // edge planes: the r planes next to each cut; interior: the rest
    if (g->lower) {
        g->edges[2 * g->nedge] = 0;
        g->edges[2 * g->nedge + 1] = std::min(r, nz);
        ++g->nedge;
    }
    if (g->upper) {
        const int lo = std::max(nz - r, g->lower ? r : 0);
        if (lo < nz) {
            g->edges[2 * g->nedge] = lo;
            g->edges[2 * g->nedge + 1] = nz;
            ++g->nedge;
        }
    }
    g->ilo = g->lower ? std::min(r, nz) : 0;
    g->ihi = g->upper ? std::max(nz - r, g->ilo) : nz;
    g->centre = g->e->lay.off(global->n[0] / 2, global->n[1] / 2, nz / 2);
    if (nccl_id) {  // (world > 1 without an id: in-process ranks, mm_cd_group_step_local)
        ncclUniqueId u;
        std::memcpy(&u, nccl_id, sizeof u);
        nccl_check(nccl().CommInitRank(&g->comm, world, u, rank), "ncclCommInitRank");
    }
    *out = g.release();
    MM_API_END
}

int mm_cd_group_destroy(mm_cd_group* g) {
    MM_API_BEGIN
    delete g;
    MM_API_END
}

int mm_cd_group_engine(mm_cd_group* g, mm_cd_engine** e) {
    MM_API_BEGIN
    need(g, "group");
    need(e, "engine");
    *e = g->e;
    MM_API_END
}

int mm_cd_group_slab(mm_cd_group* g, int* z0, int* nz) {
    MM_API_BEGIN
    need(g, "group");
    if (z0) *z0 = g->z0;
    if (nz) *nz = g->nz;
    MM_API_END
}

int mm_cd_group_step(mm_cd_group* g, float amp, const int* src_global) {
    MM_API_BEGIN
    need(g, "group");
    MM_CUDA(cudaSetDevice(g->e->device));
    if (g->world > 1 && !g->comm)
        raise(ST_NCCL, "group has no communicator (in-process ranks step with mm_cd_group_step_local)");
    g->step(amp, g->local_src(src_global), nullptr, nullptr, nullptr);
    MM_API_END
}

int mm_cd_group_step_local(mm_cd_group** groups, int n, float amp, const int* src_global) {
    MM_API_BEGIN
    need(groups, "groups");
    if (n < 1) raise(ST_INVAL, "need at least one rank");
    for (int i = 0; i < n; ++i) {
        need(groups[i], "group");
        if (groups[i]->world != n || groups[i]->rank != i)
            raise(ST_INVAL, "groups must be the ranks 0 .. n-1 of one decomposition");
        if (groups[i]->e->device != groups[0]->e->device)
            raise(ST_INVAL, "in-process ranks share one device");
    }
    MM_CUDA(cudaSetDevice(groups[0]->e->device));
    std::vector<mm_cd_group::StepArgs> args(n);
    for (int i = 0; i < n; ++i) {
        groups[i]->local_peers = groups;
        args[i] = {amp, groups[i]->local_src(src_global), nullptr, nullptr, nullptr};
    }
    try {
        for (int i = 0; i < n; ++i) groups[i]->phase1(args[i]);
        for (int i = 0; i < n; ++i) groups[i]->phase2(args[i]);
    } catch (...) {
        for (int i = 0; i < n; ++i) groups[i]->local_peers = nullptr;
        throw;
    }
    for (int i = 0; i < n; ++i) groups[i]->local_peers = nullptr;
    MM_API_END
}

int mm_cd_group_run(mm_cd_group* g, const float* amps, int nsteps, const int* src_global,
                    int record, int first_sample, float* device_ms) {
    MM_API_BEGIN
    need(g, "group");
    mm_cd_engine* e = g->e;
    MM_CUDA(cudaSetDevice(e->device));
    if (nsteps < 0) raise(ST_INVAL, "nsteps must be >= 0");
    if (nsteps == 0) return MM_OK;
    need(amps, "amps");
    if (g->world > 1 && !g->comm) raise(ST_NCCL, "group has no communicator");
    const bool rec_on = record && e->nrec > 0;
    if (rec_on && (first_sample < 0 || first_sample + nsteps > e->cap))
        raise(ST_INVAL, "recorded steps exceed the trace capacity");
    const long long so = g->local_src(src_global);
    e->amps.upload(amps, nsteps, e->stream);
    const int init[2] = {0, INT_MAX};
    MM_CUDA(cudaMemcpyAsync(e->counters.ptr, init, sizeof init, cudaMemcpyHostToDevice, e->stream));
    int* step_dev = e->counters.ptr;
    int* bad = e->counters.ptr + 1;
    struct Ev {
        cudaEvent_t a = nullptr, b = nullptr;
        ~Ev() {
            if (a) cudaEventDestroy(a);
            if (b) cudaEventDestroy(b);
        }
    } ev;
    MM_CUDA(cudaEventCreate(&ev.a));
    MM_CUDA(cudaEventCreate(&ev.b));
    MM_CUDA(cudaEventRecord(ev.a, e->stream));
    const RecParams rp{nullptr, e->rec_offs.ptr, e->traces.ptr + (size_t)first_sample * e->nrec,
                       rec_on ? e->nrec : 0, 0, bad};
    for (int s = 0; s < nsteps; ++s) g->step(0.0f, so, e->amps.ptr, step_dev, &rp);
    MM_CUDA(cudaEventRecord(ev.b, e->stream));
    MM_CUDA(cudaEventSynchronize(ev.b));
    float ms = 0;
    MM_CUDA(cudaEventElapsedTime(&ms, ev.a, ev.b));
    if (device_ms) *device_ms = ms;
    int bad_h = INT_MAX;
    MM_CUDA(cudaMemcpy(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost));
    if (bad_h != INT_MAX)  // ref: dist.cpp:222-224
        throw Error(ST_INSTABILITY,
                    "non-finite wavefield sample on rank " + std::to_string(g->rank) +
                        " at time step " + std::to_string(first_sample + bad_h),
                    first_sample + bad_h);
    MM_API_END
}

}  // extern "C"
