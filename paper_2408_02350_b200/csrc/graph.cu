// graph.cu -- one BGK step (bgk_step at a single rank) as a CUDA graph.
//
// The eager step is ~20 small launches (geometry, transport, moments, relaxation, walls); on the 2D
// workloads (sub-millisecond steps) their launch gaps and, with particle management, the host read
// of the decision counts (one stream synchronisation per step) are a visible part of the step.  Here
// the step is captured once per buffer parity and replayed with one cudaGraphLaunch.
//
// Particle management (Z28) decides on the device whether the cloud changes; applying a
// change needs the host (new N, lists, TMA maps).  The managed graph therefore has two conditional
// nodes: IF #1 (no earlier step was skipped) { neighbours; detect; decide; gate } and IF #2 (the
// decision changed nothing) { WLS, transport, moments, relaxation, walls; count the step }.  A
// change sets a sticky device flag, so that step and every graph step enqueued after it do nothing;
// graph_reconcile (called by every ABI entry that reads or changes the state) finds the flag, puts
// fcur back to the first skipped step and runs the skipped steps again -- the first of them eagerly,
// which applies the change exactly as the eager path does.  On the lattice workloads no pass changes
// anything, so no step is ever skipped.
#include <cstdlib>

#include "bgk_internal.cuh"

namespace bgk {

namespace {

__global__ void k_gate_pending(cudaGraphConditionalHandle h, const int64_t* __restrict__ flag) {
    cudaGraphSetConditional(h, flag[0] == 0 ? 1u : 0u);
}

// flag[0]: a change skipped the rest (sticky until reconciled), flag[1]: bodies run since the last
// reconcile, flag[2]: bodies run in total, flag[3]: the test hook below has fired.  skip_at >= 0
// (BGK_TEST_GRAPH_SKIP_AT, tests only) treats graph step number skip_at as a change once, so the
// skip / reconcile / re-run machinery is exercised on clouds where no pass ever changes anything.
__global__ void k_gate_changed(cudaGraphConditionalHandle h, const int64_t* __restrict__ rep, int64_t* flag,
                               int64_t skip_at) {
    bool changed = rep[7] != 0;
    if (!changed && skip_at >= 0 && flag[3] == 0 && flag[2] == skip_at) {
        changed = true;
        flag[3] = 1;
    }
    if (changed) flag[0] = 1;
    cudaGraphSetConditional(h, changed ? 0u : 1u);
}

__global__ void k_step_done(int64_t* flag) {
    flag[1] += 1;
    flag[2] += 1;
}

uint64_t mix(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
}

// everything a captured step's kernel parameters depend on, besides the buffer parity (slot)
uint64_t graph_key(const bgk_ctx* c) {
    uint64_t h = 0x42474b;
    h = mix(h, (uint64_t)c->N);
    h = mix(h, (uint64_t)c->N_int);
    h = mix(h, (uint64_t)c->N_b);
    h = mix(h, c->cloud_gen);
    h = mix(h, (uint64_t)c->geometry_valid);
    return h | 1ull;    // 0 = empty slot
}

}  // namespace

bool graph_enabled() {
    static const bool on = [] {
        const char* e = getenv("BGK_GRAPH");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

namespace {

// the part of ensure_geometry after neighbours and management (ALE: every step).  The boundary
// half of the WLS and the interpolation unions (k_wls_boundary -> k_bnd_union, small single-wave
// kernels) run on a forked branch beside the interior WLS: they write disjoint rows.
void geometry_tail(bgk_ctx* c, cudaStream_t s) {
    cudaEventRecord(c->cap_fork, s);
    cudaStreamWaitEvent(c->cap_stream3, c->cap_fork, 0);
    launch_wls_boundary(c, c->cap_stream3);
    launch_bnd_union(c, c->cap_stream3);
    launch_wls_interior(c, s);
    cudaEventRecord(c->cap_join, c->cap_stream3);
    cudaStreamWaitEvent(s, c->cap_join, 0);
}

// transport .. boundary fill with the current parity (fcur is flipped by the caller)
void phases(bgk_ctx* c, cudaStream_t s) {
    double* fn = c->f[1 - c->fcur];
    if (c->fuse2) {
        launch_transport_fused(c, c->f[c->fcur], fn, s);
    } else {
        launch_transport(c, c->f[c->fcur], fn, s);
        launch_moment_reduce(c, s);
        launch_relax(c, fn, s);
    }
    launch_boundary_interp(c, fn, s);
    launch_boundary_fill(c, fn, s);
}

// append IF(h) { body } to the capture on cs; the body is captured on bs into the node's child graph
template <typename F>
bool add_if(cudaStream_t cs, cudaStream_t bs, cudaGraphConditionalHandle h, F&& body) {
    cudaStreamCaptureStatus st;
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    if (cudaStreamGetCaptureInfo(cs, &st, nullptr, &cg, &deps, &nd) != cudaSuccess ||
        st != cudaStreamCaptureStatusActive)
        return false;
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeIf;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    if (cudaGraphAddNode(&node, cg, deps, nd, &p) != cudaSuccess) return false;
    if (cudaStreamUpdateCaptureDependencies(cs, &node, 1, cudaStreamSetCaptureDependencies) != cudaSuccess)
        return false;
    cudaGraph_t child = p.conditional.phGraph_out[0];
    if (cudaStreamBeginCaptureToGraph(bs, child, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
        cudaSuccess)
        return false;
    body(bs);
    cudaGraph_t out = nullptr;
    return cudaStreamEndCapture(bs, &out) == cudaSuccess;
}

bool capture(bgk_ctx* c, int slot) {
    if (!c->cap_stream) {
        if (cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess) return false;
        if (cudaStreamCreateWithFlags(&c->cap_stream2, cudaStreamNonBlocking) != cudaSuccess) return false;
        if (cudaStreamCreateWithFlags(&c->cap_stream3, cudaStreamNonBlocking) != cudaSuccess) return false;
        if (cudaEventCreateWithFlags(&c->cap_fork, cudaEventDisableTiming) != cudaSuccess) return false;
        if (cudaEventCreateWithFlags(&c->cap_join, cudaEventDisableTiming) != cudaSuccess) return false;
    }
    cudaStream_t cs = c->cap_stream, bs = c->cap_stream2;
    const bool managed = c->cfg.manage && c->cfg.ale;
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return false;
    bool ok = true;
    if (!managed) {
        if (c->cfg.ale) {
            launch_build_neighbors(c, cs);
            geometry_tail(c, cs);
        }
        phases(c, cs);
    } else {
        cudaStreamCaptureStatus st;
        cudaGraph_t cg = nullptr;
        ok = cudaStreamGetCaptureInfo(cs, &st, nullptr, &cg) == cudaSuccess;
        cudaGraphConditionalHandle h1 = 0, h2 = 0;
        ok = ok && cudaGraphConditionalHandleCreate(&h1, cg, 0, cudaGraphCondAssignDefault) == cudaSuccess;
        ok = ok && cudaGraphConditionalHandleCreate(&h2, cg, 0, cudaGraphCondAssignDefault) == cudaSuccess;
        if (ok) {
            k_gate_pending<<<1, 1, 0, cs>>>(h1, c->gflag);
            ok = add_if(cs, bs, h1, [&](cudaStream_t b) {
                launch_build_neighbors(c, b);
                manage_decide(c, b);
                const char* sk = getenv("BGK_TEST_GRAPH_SKIP_AT");
                k_gate_changed<<<1, 1, 0, b>>>(h2, c->mg.rep, c->gflag, sk ? atoll(sk) : -1);
            });
        }
        ok = ok && add_if(cs, bs, h2, [&](cudaStream_t b) {
            geometry_tail(c, b);
            phases(c, b);
            k_step_done<<<1, 1, 0, b>>>(c->gflag);
        });
    }
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(cs, &g);
    ok = ok && e == cudaSuccess && g != nullptr;
    if (ok) {
        if (c->gexec[slot]) cudaGraphExecDestroy(c->gexec[slot]);
        c->gexec[slot] = nullptr;
        ok = cudaGraphInstantiate(&c->gexec[slot], g, 0) == cudaSuccess;
    }
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();   // a failed capture leaves no sticky error: the eager path takes over
    return ok;
}

}  // namespace

bool graph_step(bgk_ctx* c, cudaStream_t s) {
    if (!graph_enabled() || !c->graph_ok || c->ncol != c->ncol_g) return false;
    cudaStreamCaptureStatus cst;
    if (cudaStreamIsCapturing(s, &cst) != cudaSuccess || cst != cudaStreamCaptureStatusNone) return false;
    if (!c->cfg.ale && !c->geometry_valid) return false;     // fixed cloud: first step builds it eagerly
    if (c->force_eager > 0) {
        --c->force_eager;
        return false;
    }
    const uint64_t key = graph_key(c);
    const int slot = c->fcur;
    if (c->gkey[slot] != key) {
        // capture only after one eager step with this key: first-use kernel attributes are set, and a
        // one-off step (e.g. right after a management change) does not pay for a capture
        if (c->eager_key != key) {
            c->eager_key = key;
            return false;
        }
        if (!capture(c, slot)) {
            c->graph_ok = false;
            return false;
        }
        c->gkey[slot] = key;
        ++c->gstat[1];
    }
    if (c->cfg.manage && c->cfg.ale) {
        if (c->gsteps == 0) c->gfcur0 = c->fcur;
        ++c->gsteps;
    }
    if (cudaGraphLaunch(c->gexec[slot], s) != cudaSuccess) {
        cudaGetLastError();
        c->graph_ok = false;
        if (c->cfg.manage && c->cfg.ale) --c->gsteps;
        return false;
    }
    c->gstream = s;
    c->fcur = 1 - c->fcur;
    ++c->gstat[0];
    return true;
}

bgk_status graph_reconcile(bgk_ctx* c, cudaStream_t s) {
    if (c->gsteps == 0) return BGK_OK;
    const int64_t n = c->gsteps;
    c->gsteps = 0;
    int64_t fl[2] = {0, 0};     // flag[0], flag[1]; flag[2], flag[3] persist
    int64_t rep[8];
    cudaError_t e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaMemcpy(fl, c->gflag, sizeof(fl), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(rep, c->mg.rep, sizeof(rep), cudaMemcpyDeviceToHost);
    const int64_t zero[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpy(c->gflag, zero, sizeof(zero), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return BGK_E_CUDA;
    for (int r = 0; r < 6; ++r) c->mg_report[r] = rep[r];
    if (fl[0] == 0) return BGK_OK;                      // every enqueued step ran
    const int64_t done = fl[1];
    c->gstat[2] += n - done;
    c->fcur = (int)((c->gfcur0 + done) & 1);            // the state is the start of step `done`
    c->eager_key = 0;
    c->force_eager = 1;
    // the skipped steps again: the first eagerly (it applies the change), the rest through bgk_step
    bgk_status st = bgk_step(c, 1, reinterpret_cast<bgk_stream>(s));
    if (st == BGK_OK && n - done - 1 > 0) st = bgk_step(c, (int)(n - done - 1), reinterpret_cast<bgk_stream>(s));
    if (st != BGK_OK) return st;
    return graph_reconcile(c, s);
}

}  // namespace bgk

extern "C" bgk_status bgk_graph_info(bgk_ctx* c, int64_t* info) {
    if (!c || !info) return BGK_E_INVALID_ARG;
    info[0] = (bgk::graph_enabled() && c->graph_ok) ? 1 : 0;
    info[1] = c->gstat[0];
    info[2] = c->gstat[1];
    info[3] = c->gstat[2];
    return BGK_OK;
}

namespace bgk {

void graph_release(bgk_ctx* c) {
    if (c->gstat[0] > 0) cudaStreamSynchronize(c->gstream);   // graph launches still in flight
    for (int b = 0; b < 2; ++b)
        if (c->gexec[b]) cudaGraphExecDestroy(c->gexec[b]);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    if (c->cap_stream2) cudaStreamDestroy(c->cap_stream2);
    if (c->cap_stream3) cudaStreamDestroy(c->cap_stream3);
    if (c->cap_fork) cudaEventDestroy(c->cap_fork);
    if (c->cap_join) cudaEventDestroy(c->cap_join);
}

}  // namespace bgk
