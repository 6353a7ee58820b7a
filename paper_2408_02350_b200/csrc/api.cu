// api.cu -- the C ABI of include/bgk.h: context, workspace carving, launch
// sequence of one step (split into the three phases a velocity-sharded run
// interleaves with its two all-reduces), copies and error reporting.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "bgk_internal.cuh"

using namespace bgk;

namespace {

constexpr const char* kVersion = "bgk_b200 0.1.0 (sm_100a, fp64)";

struct Carver {
    char* base;
    size_t off = 0;
    bool dry;
    template <typename T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T* p = dry ? nullptr : reinterpret_cast<T*>(base + off);
        off += sizeof(T) * std::max<size_t>(count, 1);
        return p;
    }
};

// x == NULL at bgk_init_cloud: the regular cavity lattice, n = L/dx + 1 points
// per axis, index = ix + n iy (+ n^2 iz), coordinates i dx with the last one exactly L; points on
// a face are boundary particles of the lowest wall id they lie on (1: x=0, 2: x=L, 3: y=0, ...).
bool make_lattice(int d, double L, double dx, int64_t N, std::vector<double>& x, std::vector<int8_t>& kind) {
    const int64_t n = (int64_t)std::llround(L / dx) + 1;
    int64_t nn = 1;
    for (int a = 0; a < d; ++a) nn *= n;
    if (n < 3 || nn != N) return false;
    for (int64_t i = 0; i < N; ++i) {
        int64_t r = i;
        int8_t k = 0;
        for (int a = 0; a < d; ++a) {
            const int64_t ia = r % n;
            r /= n;
            x[i * d + a] = ia == n - 1 ? L : (double)ia * dx;
            const int8_t wid = ia == 0 ? (int8_t)(2 * a + 1) : (ia == n - 1 ? (int8_t)(2 * a + 2) : 0);
            if (wid && (k == 0 || wid < k)) k = wid;
        }
        kind[i] = k;
    }
    return true;
}

bool valid_cfg(const bgk_config* c, int64_t N) {
    if (!c || N < 1) return false;
    if (c->dims != 2 && c->dims != 3) return false;
    if (c->Nv < 2 || c->Nv + 1 > 64) return false;   // odd Nv allowed: the paper's Figs. 6-7 use Nv = 15
    if (std::isnan(c->vmax) || !(c->L > 0.0) || !(c->h > 0.0) || !(c->h2 > 0.0) || !(c->dt >= 0.0)) return false;
    if (!(c->R > 0.0) || !(c->kb > 0.0) || !(c->dmol > 0.0) || !(c->T_wall > 0.0) || !(c->alpha_w > 0.0)) return false;
    if (N > (int64_t)INT32_MAX || c->max_particles > (int64_t)INT32_MAX) return false;
    if (c->manage != 0 && c->manage != 1) return false;
    if (c->staging != 0 && c->staging != 1) return false;
    if (c->wls_order < 0 || c->wls_order > 2) return false;
    return true;
}

// geometry + mapping that only depends on the configuration and N
void derive(bgk_ctx* c, const bgk_config* cfg, int64_t N) {
    c->cfg = *cfg;
    if (!(c->cfg.vmax > 0.0)) {   // v_max = |U_wall| + 4 sqrt(R T_wall)
        const double* u = cfg->U_lid;
        c->cfg.vmax = std::sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]) + 4.0 * std::sqrt(cfg->R * cfg->T_wall);
    }
    cfg = &c->cfg;
    c->d = cfg->dims;
    c->nv = c->d == 2 ? 2 : 1;
    c->n1 = cfg->Nv + 1;
    c->ncol_g = c->d == 2 ? c->n1 : c->n1 * c->n1;
    if (cfg->col_begin == 0 && cfg->col_end == 0) {
        c->c0 = 0;
        c->c1 = c->ncol_g;
    } else {
        c->c0 = cfg->col_begin;
        c->c1 = cfg->col_end;
    }
    c->ncol = c->c1 - c->c0;
    c->N = N;
    c->Ncap = std::max<int64_t>(N, cfg->max_particles);
    c->Kloc = (int64_t)c->n1 * c->ncol;
    // 3D row stride padded to a multiple of 16 doubles (128 B): every 256-B box row of a column group
    // then starts on a cache line and covers exactly 8 L2 sectors (C5 transport: 75.7 ms at 16-B
    // rows, 73.4 at 32 B, 72.8 at 64 B, 71.4 at 128 B; profiles/r01_tuning.md); BGK_NCS_ALIGN overrides.
    // 2D rows stay unpadded (128-B padding measured no gain on C2/C3, profiles/r01_tuning.md).
    {
        static const int al = [] {
            const char* e = getenv("BGK_NCS_ALIGN");
            const int v = e ? atoi(e) : 16;
            return (v == 2 || v == 4 || v == 8 || v == 16) ? v : 16;
        }();
        c->ncs = c->d == 3 ? (c->ncol + al - 1) / al * al : c->ncol;
    }
    c->Ks = (int64_t)c->n1 * c->ncs;
    c->RS = c->Ks * c->nv;
    c->max_nb = cfg->max_neighbors > 0 ? cfg->max_neighbors : (c->d == 2 ? 96 : 256);
    c->cap = c->Ncap * (int64_t)c->max_nb;
    int nc = (int)std::floor(cfg->L / cfg->h);
    nc = std::max(1, std::min(nc, cfg->dims == 3 ? 1024 : kMaxCellsPerAxis));
    while (nc > 1 && cfg->L / nc < cfg->h * (1.0 + 1e-12)) --nc;   // cell edge strictly >= h
    int pw = 1;                                  // Morton cell codes span a power-of-two box
    while (pw < nc) pw <<= 1;
    c->ncell = 1;
    for (int a = 0; a < 3; ++a) {
        c->nc[a] = a < c->d ? nc : 1;
        c->edge[a] = cfg->L / nc;
        c->ncell *= a < c->d ? pw : 1;
    }
    c->dv = 2.0 * cfg->vmax / cfg->Nv;
    c->vmin = -cfg->vmax;
    c->wls_order = cfg->wls_order == 2 ? 2 : 1;
    c->PD = (c->d == 2 ? 4 : 10) + (c->wls_order == 2 ? 2 : 0);
    c->R = transport_rows_per_thread(c->d, c->n1);
    c->nchunk = (c->n1 + c->R - 1) / c->R;   // the last chunk may be ragged
    c->ncg = (c->ncol + 31) / 32;           // a warp = (chunk, 32-column group): one TMA box per neighbour
    // 2D, 33 columns (N_v = 32): a 32-lane group for ONE column would idle 31 lanes -- the box of
    // the single group carries column 32 as well and lanes 0..R-1 update its R nodes of the chunk
    // (k_transport XC = 1); instantiated for R = 17, 13, 11, 9, first order
    c->xc = (c->d == 2 && c->ncol == 33 && (c->R == 17 || c->R == 13 || c->R == 11 || c->R == 9) &&
             c->wls_order == 1)
                ? 1
                : 0;
    if (c->xc) c->ncg = 1;
    {
        const char* e = getenv("BGK_FUSE");
        c->fuse2 = (c->xc && c->R == 11 && c->n1 == 33 && c->ncol == c->ncol_g && !(e && atoi(e) == 0)) ? 1 : 0;
    }
    c->nwpp = c->nchunk * c->ncg;
    // 3D: a last column group of at most 16 columns (e.g. 78-79 columns per rank at P = 8 on C5) runs
    // folded -- 16 columns x two halves of v_1 in one warp -- instead of a full-width pass with half
    // the lanes idle (k_transport FD = 1); needs the whole v_1 axis in one chunk and n1 <= 2 kFoldR
    {
        const char* e = getenv("BGK_FOLD");
        const int wl = c->ncol - 32 * (c->ncg - 1);
        c->fold = (c->d == 3 && c->wls_order == 1 && c->nchunk == 1 && c->n1 <= 2 * kFoldR && wl >= 1 &&
                   wl <= 16 && !(e && atoi(e) == 0))
                      ? 1
                      : 0;
    }
    c->nslots = c->nwpp * 32;
    // fixed-cloud lattice rows (SURVEY §8(d) "the one lever"): partial slots sized for both mappings
    {
        const char* e = getenv("BGK_TRANSPORT_ROWS");
        c->rows_on = !cfg->ale && c->d == 3 && c->wls_order == 1 && c->ncol == c->ncol_g &&
                     c->Ncap < (1 << 23) && c->max_nb <= 256 &&
                     !(e && atoi(e) == 0);
        c->rows_nchunk = (c->n1 + kRowsR - 1) / kRowsR;
        if (c->rows_on) c->nwpp = std::max(c->nchunk, c->rows_nchunk) * c->ncg;
    }
    c->bnd_chunk = 256;
    // boundary interpolation chunks: 3D the tile kernel's per-wall plan of incoming nodes (bnd_plan),
    // 2D k_bnd_interp_t's 256 threads x 2 stored nodes
    if (c->d == 3) c->bnd_nch = std::max(1, bnd_plan(c, nullptr, nullptr, nullptr, c->bnd_nchw));
    else c->bnd_nch = (int)((c->Ks + 511) / 512);
}

// particle-management scratch (only when cfg.manage): decision arrays over the capacity, the
// gathered per-particle arrays, and the interpolation stencils of up to kManageMaxNew new particles
void carve_manage(bgk_ctx* c, Carver& k) {
    const bool on = c->cfg.manage != 0;
    const int64_t N = on ? c->Ncap : 1;
    const int d = c->d;
    const int64_t nn = on ? kManageMaxNew : 1;
    Manage& m = c->mg;
    m.flag = k.take<uint8_t>(N);
    m.status = k.take<int32_t>(N);
    m.map = k.take<int32_t>(N);
    m.x = k.take<double>(N * d);
    m.W = k.take<double>(N * d);
    m.macro = k.take<double>(N * (d + 2));
    m.kind = k.take<int8_t>(N);
    m.pos = k.take<double>(nn * d);
    m.nW = k.take<double>(nn * d);
    m.nM = k.take<double>(nn * (d + 2));
    m.dst = k.take<int32_t>(nn);
    m.sm = k.take<int32_t>(nn);
    m.sidx = k.take<int32_t>(nn * c->max_nb);
    m.sc = k.take<double>(nn * c->max_nb);
    m.rep = k.take<int64_t>(8);
    m.counts = k.take<int32_t>(4);
}

size_t carve(bgk_ctx* c, char* base, bool dry) {
    Carver k{base, 0, dry};
    const int64_t N = c->Ncap;   // every per-particle buffer is sized for the capacity
    const int d = c->d;
    c->x = k.take<double>(N * d);
    c->kind = k.take<int8_t>(N);
    c->interior = k.take<int32_t>(N);
    c->boundary = k.take<int32_t>(N);
    c->W = k.take<double>(N * d);
    c->macro = k.take<double>(N * (d + 2));
    c->f[0] = k.take<double>((size_t)N * c->RS);
    c->f[1] = k.take<double>((size_t)N * c->RS);
    c->partials = k.take<double>((size_t)N * c->nwpp * kPM);
    c->sums = k.take<double>((size_t)N * kPM);
    c->wallpart = k.take<double>((size_t)N * c->bnd_nch);
    c->wallnum = k.take<double>(N);
    c->Mw = k.take<double>((size_t)2 * d * c->RS);
    c->wall_den = k.take<double>(2 * d);
    c->outbuf = k.take<double>(N * (d + 2));
    c->err = k.take<int64_t>(4);
    c->gflag = k.take<int64_t>(4);
    c->stab = k.take<unsigned long long>(1);
    c->scan_tmp = k.take<int64_t>(1024);
    c->blk_tmp = k.take<int32_t>(1024);
    c->g.cell_of = k.take<int32_t>(N);
    c->g.cell_cnt = k.take<int32_t>(c->ncell);
    c->g.cell_start = k.take<int32_t>(c->ncell + 1);
    c->g.cell_fill = k.take<int32_t>(c->ncell);
    c->g.cell_pts = k.take<int32_t>(N);
    c->g.nb_cnt = k.take<int32_t>(N);
    c->g.nb_off = k.take<int64_t>(N + 1);
    c->g.nb_idx = k.take<int32_t>(c->cap);
    c->g.S = k.take<double>(N * d * d);
    c->g.P = k.take<double>((size_t)c->cap * c->PD);
    c->g.cw = k.take<double>(c->cap);
    c->g.bidx = k.take<int32_t>(c->cap);
    c->g.bcw = k.take<double>(c->cap);
    c->g.bcnt = k.take<int32_t>(N);
    c->g.order = k.take<int32_t>(N);
    carve_manage(c, k);
    c->stage = k.take<double>(c->cfg.staging ? (size_t)N * c->nv * c->Kloc : 1);
    {
        // boundary interpolation groups: 3D face tiles of up to kBndTile members (install_lists; at most
        // N / 8 + 64 groups, else runs of kBndTile), 2D 4 consecutive boundary particles
        c->bnd_g = c->d == 3 ? kBndTile : 4;
        c->bu_cap = std::min(c->bnd_g * c->max_nb, 512);   // union rows per group (CAPACITY beyond)
        c->bg_max = c->d == 3 ? N / 8 + 64 : N / c->bnd_g + 1;
        const size_t ng = (size_t)c->bg_max;
        c->bg_off = k.take<int32_t>(ng + 1);
        c->bu_j = k.take<int32_t>(ng * c->bu_cap);
        c->bu_w = k.take<double>(ng * c->bu_cap * c->bnd_g);
        c->bu_n = k.take<int32_t>(ng);
        const size_t nt = c->d == 3 ? (size_t)2 * d * c->bnd_nch : 1;
        c->bnd_chunks = k.take<BndChunk>(nt);
        c->bnd_act_t = k.take<int32_t>(nt * (c->d == 3 ? kBndAct : 1));
        c->bnd_act_s = k.take<int32_t>(nt * (c->d == 3 ? kBndAct : 1));
    }
    c->rows_p0 = k.take<int32_t>(c->rows_on ? (size_t)N / kRowsG + 1 : 1);
    c->rows_stride = k.take<int32_t>(c->rows_on ? (size_t)N / kRowsG + 1 : 1);
    c->rows_perm = k.take<int16_t>(c->rows_on ? ((size_t)N / kRowsG + 1) * 256 : 1);
    c->order_rest = k.take<int32_t>(c->rows_on ? (size_t)N : 1);
    c->tile_org = k.take<int32_t>(c->rows_on ? ((size_t)N / 512 + 1) * 3 : 1);
    c->ctab = k.take<double>(c->rows_on ? (size_t)123 * c->Ks : 1);
    return k.off + 256;
}

bgk_status cuda_fail(bgk_ctx* c, cudaError_t e) {
    if (c) {
        std::snprintf(c->msg, sizeof(c->msg), "CUDA error: %s", cudaGetErrorString(e));
        c->bad = -1;
    }
    return BGK_E_CUDA;
}

bgk_status check_launch(bgk_ctx* c) {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BGK_OK : cuda_fail(c, e);
}

const char* code_msg(int code) {
    switch (code) {
        case BGK_E_CAPACITY: return "neighbour capacity exceeded (max_neighbors)";
        case BGK_E_DEFICIENT_STENCIL: return "deficient WLS stencil (< dims+2 neighbours or ill-conditioned)";
        case BGK_E_DEGENERATE_STATE: return "degenerate state (rho <= 0 or T <= 1e-12)";
        case BGK_E_OUT_OF_DOMAIN: return "particle outside [0, L]^dims";
        case BGK_E_WALL: return "diffuse-reflection denominator <= 0";
        default: return "error";
    }
}

// synchronise the stream and surface (then clear) a latched device error
bgk_status sync_check(bgk_ctx* c, cudaStream_t s) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(c, e);
    unsigned long long h = 0;
    e = cudaMemcpy(&h, c->err, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(c, e);
    if (h != 0) {                       // latch_error's packed word: code << 56 | particle
        const int code = (int)(h >> 56);
        const unsigned long long part = h & kErrNoParticle;
        std::snprintf(c->msg, sizeof(c->msg), "%s", code_msg(code));
        c->bad = part == kErrNoParticle ? -1 : (int64_t)part;
        const unsigned long long reset = 0;
        cudaMemcpy(c->err, &reset, sizeof(reset), cudaMemcpyHostToDevice);
        return (bgk_status)code;
    }
    return BGK_OK;
}

cudaStream_t S(bgk_stream s) { return reinterpret_cast<cudaStream_t>(s); }

// settle graph steps that a particle-management change skipped (graph.cu) before the state is used
#define BGK_RECONCILE(c, s)                                         \
    do {                                                            \
        const bgk_status rc_ = bgk::graph_reconcile((c), (s));      \
        if (rc_ != BGK_OK) return rc_;                              \
    } while (0)

}  // namespace

// interior / boundary lists from host kinds and positions (boundary particles sorted by
// (wall, z, y, x) so face neighbours are adjacent), counts, and the TMA maps (their outer
// extent is N).  Synchronous host->device copies (the host vectors die on return).
bgk_status bgk::install_lists(bgk_ctx* c, const int8_t* hk, const double* hx, cudaStream_t s) {
    const int64_t N = c->N;
    const int d = c->d;
    std::vector<int32_t> in, bd;
    for (int64_t i = 0; i < N; ++i) (hk[i] == 0 ? in : bd).push_back((int32_t)i);
    std::stable_sort(bd.begin(), bd.end(), [&](int32_t a, int32_t b) {
        if (hk[a] != hk[b]) return hk[a] < hk[b];
        for (int q = d - 1; q >= 0; --q)
            if (hx[(int64_t)a * d + q] != hx[(int64_t)b * d + q]) return hx[(int64_t)a * d + q] < hx[(int64_t)b * d + q];
        return a < b;
    });
    c->N_int = (int64_t)in.size();
    c->N_b = (int64_t)bd.size();
    // 3D: face tiles for the boundary interpolation.  Within a wall the order above is (slow, fast)
    // in-plane (x-walls (z, y), y-walls (z, x), z-walls (y, x)); rows are runs of one slow coordinate,
    // a member's tile is (row / 4, position in its row / 4) -- 4 x 4 points on a lattice face -- and
    // the wall's members are re-ordered tile by tile (stable).  A group is a tile's run, split into
    // runs of kBndTile; if that gives more than bg_max groups, plain runs of kBndTile per wall.
    std::vector<int32_t> goff{0};
    if (d == 3) {
        const double tol = 1e-9 * c->cfg.L;
        std::vector<int32_t> tiled;
        tiled.reserve(bd.size());
        for (size_t i = 0; i < bd.size();) {
            size_t j = i;
            while (j < bd.size() && hk[bd[j]] == hk[bd[i]]) ++j;
            const int ax = (hk[bd[i]] - 1) / 2, sa = ax == 2 ? 1 : 2;
            std::vector<std::array<int64_t, 2>> key;
            int64_t rs = 0, rf = 0;
            for (size_t q = i; q < j; ++q) {
                if (q > i) {
                    if (std::fabs(hx[(int64_t)bd[q] * d + sa] - hx[(int64_t)bd[q - 1] * d + sa]) > tol) {
                        ++rs;
                        rf = 0;
                    } else {
                        ++rf;
                    }
                }
                key.push_back({(rs / 4) * (int64_t)bd.size() + rf / 4, (int64_t)q});
            }
            std::stable_sort(key.begin(), key.end(),
                             [](const std::array<int64_t, 2>& a, const std::array<int64_t, 2>& b) { return a[0] < b[0]; });
            for (size_t q = 0; q < key.size(); ++q) {
                tiled.push_back(bd[key[q][1]]);
                const int run = (int)(tiled.size() - goff.back());
                const bool last = q + 1 == key.size() || key[q + 1][0] != key[q][0];
                if (last || run == kBndTile) goff.push_back((int32_t)tiled.size());
            }
            i = j;
        }
        if ((int64_t)goff.size() - 1 > c->bg_max) {          // fall back to runs of kBndTile per wall
            goff.assign(1, 0);
            for (size_t i = 0; i < bd.size();) {
                size_t j = i;
                while (j < bd.size() && hk[bd[j]] == hk[bd[i]]) ++j;
                for (size_t q = i; q < j; q += kBndTile) goff.push_back((int32_t)std::min(j, q + kBndTile));
                i = j;
            }
        } else {
            bd.swap(tiled);
        }
        c->n_bg = (int64_t)goff.size() - 1;
    }
    if (!make_tensor_maps(c)) return BGK_E_CUDA;
    cudaError_t e = cudaSuccess;
    if (!in.empty()) e = cudaMemcpyAsync(c->interior, in.data(), sizeof(int32_t) * in.size(), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && !bd.empty())
        e = cudaMemcpyAsync(c->boundary, bd.data(), sizeof(int32_t) * bd.size(), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && d == 3)
        e = cudaMemcpyAsync(c->bg_off, goff.data(), sizeof(int32_t) * goff.size(), cudaMemcpyHostToDevice, s);
    // interior ids also serve as the initial processing order (the neighbour build re-sorts it)
    if (e == cudaSuccess && !in.empty())
        e = cudaMemcpyAsync(c->g.order, in.data(), sizeof(int32_t) * in.size(), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return e == cudaSuccess ? BGK_OK : cuda_fail(c, e);
}

namespace {

bgk_status ensure_geometry(bgk_ctx* c, cudaStream_t s) {
    if (c->cfg.ale || !c->geometry_valid) {
        launch_build_neighbors(c, s);
        if (c->cfg.manage && c->cfg.ale) {        // particle management on the step-start cloud (Z28)
            bool changed = false;
            bgk_status st = manage_pass(c, s, &changed);
            if (st != BGK_OK) return st;
            if (changed) launch_build_neighbors(c, s);
        }
        launch_wls(c, s);
        launch_bnd_union(c, s);
        c->geometry_valid = true;
        c->rows_built = false;
        if (c->rows_on) {                         // fixed cloud: detect the lattice rows once
            bgk_status st = build_rows(c, s);
            if (st != BGK_OK) return st;
        }
    }
    return BGK_OK;
}

bgk_status copy_out(bgk_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t s) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s);
    if (e != cudaSuccess) return cuda_fail(c, e);
    return BGK_OK;
}

}  // namespace

extern "C" {

const char* bgk_version(void) { return kVersion; }

bgk_status bgk_workspace_size(const bgk_config* cfg, int64_t N, size_t* bytes) {
    if (!valid_cfg(cfg, N) || !bytes) return BGK_E_INVALID_ARG;
    bgk_ctx tmp{};
    derive(&tmp, cfg, N);
    if (tmp.c0 < 0 || tmp.c1 > tmp.ncol_g || tmp.c0 >= tmp.c1) return BGK_E_INVALID_ARG;
    *bytes = carve(&tmp, nullptr, true);
    return BGK_OK;
}

bgk_status bgk_init_cloud(const bgk_config* cfg, const double* x, const int8_t* kind, const double* macro0,
                          int64_t N, void* workspace, size_t ws_bytes, bgk_stream stream, bgk_ctx** out) {
    if (!out || !workspace || (!x) != (!kind)) return BGK_E_INVALID_ARG;
    *out = nullptr;
    size_t need = 0;
    if (bgk_workspace_size(cfg, N, &need) != BGK_OK || ws_bytes < need) return BGK_E_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(workspace) % 16) return BGK_E_INVALID_ARG;
    bgk_ctx* c = new (std::nothrow) bgk_ctx{};
    if (!c) return BGK_E_INVALID_ARG;
    derive(c, cfg, N);
    carve(c, reinterpret_cast<char*>(workspace), false);
    c->bad = -1;
    c->fcur = 0;
    c->geometry_valid = false;
    cudaStream_t s = S(stream);
    // kinds and positions on the host to build the interior / boundary lists
    std::vector<int8_t> hk(N);
    std::vector<double> hx(N * c->d);
    cudaError_t e = cudaSuccess;
    if (x) {
        e = cudaMemcpy(hk.data(), kind, N, cudaMemcpyDefault);
        if (e == cudaSuccess) e = cudaMemcpy(hx.data(), x, sizeof(double) * N * c->d, cudaMemcpyDefault);
        if (e != cudaSuccess) { bgk_status st = cuda_fail(c, e); delete c; return st; }
    } else if (!make_lattice(c->d, cfg->L, cfg->dx, N, hx, hk)) {
        delete c;
        return BGK_E_INVALID_ARG;
    }
    for (int64_t i = 0; i < N; ++i)
        if (hk[i] < 0 || hk[i] > 2 * c->d) { delete c; return BGK_E_INVALID_ARG; }
    {
        bgk_status st = install_lists(c, hk.data(), hx.data(), s);
        if (st == BGK_OK) st = upload_bnd_plan(c, s);
        if (st != BGK_OK) { delete c; return st; }
    }
    const int64_t reset[4] = {0, 0, 0, 0};
    cudaMemcpyAsync(c->err, reset, sizeof(reset), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(c->gflag, reset, 4 * sizeof(int64_t), cudaMemcpyHostToDevice, s);
    c->graph_ok = true;
    // padding columns stay zero forever (TMA boxes of the last column group read them): both
    // buffers are cleared over the whole capacity, so rows that management appends past the
    // initial N start with zero padding too (the kernels only ever write valid columns)
    cudaMemsetAsync(c->f[0], 0, sizeof(double) * c->Ncap * c->RS, s);
    cudaMemsetAsync(c->f[1], 0, sizeof(double) * c->Ncap * c->RS, s);
    cudaMemsetAsync(c->stab, 0, sizeof(unsigned long long), s);
    // rank-local sums exchanged by the caller (all-reduce): defined for every slot, boundary rows too
    cudaMemsetAsync(c->sums, 0, sizeof(double) * c->Ncap * kPM, s);
    cudaMemsetAsync(c->wallnum, 0, sizeof(double) * c->Ncap, s);
    cudaMemcpyAsync(c->x, hx.data(), sizeof(double) * N * c->d, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(c->kind, hk.data(), N, cudaMemcpyHostToDevice, s);
    const double* m0 = nullptr;
    if (macro0) {
        cudaMemcpyAsync(c->outbuf, macro0, sizeof(double) * N * (c->d + 2), cudaMemcpyDefault, s);
        m0 = c->outbuf;
    }
    if (c->cfg.staging) {
        cudaEventCreateWithFlags(&c->ev_staged, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&c->ev_consumed, cudaEventDisableTiming);
        cudaEventRecord(c->ev_consumed, s);
    }
    launch_check_domain(c, s);
    launch_wall_tables(c, s);
    launch_init_f(c, m0, s);
    bgk_status st = check_launch(c);
    if (st == BGK_OK) st = sync_check(c, s);
    if (st != BGK_OK && st != BGK_E_OUT_OF_DOMAIN && st != BGK_E_WALL) { delete c; return st; }
    if (st != BGK_OK) { delete c; return st; }
    *out = c;
    return BGK_OK;
}

bgk_status bgk_build_neighbors(bgk_ctx* c, int64_t* offsets, int32_t* idx, int64_t cap, int64_t* needed,
                               bgk_stream stream) {
    if (!c) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    cudaStream_t s = S(stream);
    launch_build_neighbors(c, s);
    c->geometry_valid = false;
    bgk_status st = check_launch(c);
    if (st == BGK_OK) st = sync_check(c, s);
    int64_t nnz = 0;
    cudaMemcpy(&nnz, c->g.nb_off + c->N, sizeof(int64_t), cudaMemcpyDeviceToHost);
    c->nnz_last = nnz;
    if (needed) *needed = nnz;
    if (st != BGK_OK) return st;
    if (offsets) {
        if (idx && nnz > cap) {
            std::snprintf(c->msg, sizeof(c->msg), "idx capacity %lld < needed %lld", (long long)cap, (long long)nnz);
            return BGK_E_CAPACITY;
        }
        if ((st = copy_out(c, offsets, c->g.nb_off, sizeof(int64_t) * (c->N + 1), s)) != BGK_OK) return st;
        if (idx && nnz && (st = copy_out(c, idx, c->g.nb_idx, sizeof(int32_t) * nnz, s)) != BGK_OK) return st;
        return sync_check(c, s);
    }
    return BGK_OK;
}

bgk_status bgk_wls_coeffs(bgk_ctx* c, bgk_stream stream) {
    if (!c) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    cudaStream_t s = S(stream);
    launch_wls(c, s);
    bgk_status st = check_launch(c);
    if (st == BGK_OK) st = sync_check(c, s);
    c->geometry_valid = false;   // the next step rebuilds the full geometry (interpolation groups, rows)
    return st;
}

bgk_status bgk_get_wls(bgk_ctx* c, double* Sout, double* rot, double* frames, double* cw, bgk_stream stream) {
    if (!c) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    cudaStream_t s = S(stream);
    const int d = c->d;
    bgk_status st = sync_check(c, s);        // in-flight geometry work finishes before nnz is read
    if (st != BGK_OK) return st;
    int64_t nnz = 0;
    cudaMemcpy(&nnz, c->g.nb_off + c->N, sizeof(int64_t), cudaMemcpyDeviceToHost);
    if (Sout && (st = copy_out(c, Sout, c->g.S, sizeof(double) * c->N * d * d, s)) != BGK_OK) return st;
    if (cw && nnz && (st = copy_out(c, cw, c->g.cw, sizeof(double) * nnz, s)) != BGK_OK) return st;
    if (rot || frames) {
        // scratch: the idle f buffer, or (tiny velocity grids) a temporary stream-ordered allocation
        double* scratch = c->f[1 - c->fcur];
        double* tmp = nullptr;
        const size_t need = (size_t)nnz * (d + d * d);
        if (need > (size_t)c->N * c->RS) {
            cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(double) * need, s);
            if (e != cudaSuccess) return cuda_fail(c, e);
            scratch = tmp;
        }
        double* r = scratch;
        double* fr = scratch + (size_t)nnz * d;
        cudaMemsetAsync(scratch, 0, sizeof(double) * nnz * (d + d * d), s);
        launch_wls_export(c, r, fr, s);
        if ((st = check_launch(c)) != BGK_OK) return st;
        if (rot && nnz && (st = copy_out(c, rot, r, sizeof(double) * nnz * d, s)) != BGK_OK) return st;
        if (frames && nnz && (st = copy_out(c, frames, fr, sizeof(double) * nnz * d * d, s)) != BGK_OK) return st;
        if (tmp) cudaFreeAsync(tmp, s);
    }
    return sync_check(c, s);
}

bgk_status bgk_run_phase(bgk_ctx* c, bgk_phase phase, bgk_stream stream) {
    if (!c) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    cudaStream_t s = S(stream);
    double* fn = c->f[1 - c->fcur];
    switch (phase) {
        case BGK_PHASE_GEOMETRY: {
            bgk_status st = ensure_geometry(c, s);
            if (st != BGK_OK) return st;
            break;
        }
        case BGK_PHASE_TRANSPORT: launch_transport(c, c->f[c->fcur], fn, s); break;
        case BGK_PHASE_MOMENT_SUMS: launch_moment_reduce(c, s); break;
        case BGK_PHASE_RELAX: launch_relax(c, fn, s); break;
        case BGK_PHASE_BOUNDARY_INTERP: launch_boundary_interp(c, fn, s); break;
        case BGK_PHASE_BOUNDARY_FILL:
            launch_boundary_fill(c, fn, s);
            c->fcur = 1 - c->fcur;
            break;
        default: return BGK_E_INVALID_ARG;
    }
    return check_launch(c);
}

bgk_status bgk_step_transport(bgk_ctx* c, bgk_stream stream) {
    bgk_status st;
    if ((st = bgk_run_phase(c, BGK_PHASE_GEOMETRY, stream)) != BGK_OK) return st;
    if ((st = bgk_run_phase(c, BGK_PHASE_TRANSPORT, stream)) != BGK_OK) return st;
    return bgk_run_phase(c, BGK_PHASE_MOMENT_SUMS, stream);
}

bgk_status bgk_step_relax(bgk_ctx* c, bgk_stream stream) {
    bgk_status st;
    if ((st = bgk_run_phase(c, BGK_PHASE_RELAX, stream)) != BGK_OK) return st;
    return bgk_run_phase(c, BGK_PHASE_BOUNDARY_INTERP, stream);
}

bgk_status bgk_step_boundary(bgk_ctx* c, bgk_stream stream) {
    return bgk_run_phase(c, BGK_PHASE_BOUNDARY_FILL, stream);
}

bgk_status bgk_step(bgk_ctx* c, int n_steps, bgk_stream stream) {
    if (!c || n_steps < 0) return BGK_E_INVALID_ARG;
    if (c->ncol != c->ncol_g) return BGK_E_INVALID_ARG;   // sharded runs use the split phases
    for (int n = 0; n < n_steps; ++n) {
        if (graph_step(c, S(stream))) continue;         // the whole step as one graph launch (graph.cu)
        bgk_status st;
        if (c->fuse2) {                                  // 2D XC: transport + relaxation in one kernel
            if ((st = bgk_run_phase(c, BGK_PHASE_GEOMETRY, stream)) != BGK_OK) return st;
            launch_transport_fused(c, c->f[c->fcur], c->f[1 - c->fcur], S(stream));
            if ((st = check_launch(c)) != BGK_OK) return st;
            if ((st = bgk_run_phase(c, BGK_PHASE_BOUNDARY_INTERP, stream)) != BGK_OK) return st;
        } else {
            if ((st = bgk_step_transport(c, stream)) != BGK_OK) return st;
            if ((st = bgk_step_relax(c, stream)) != BGK_OK) return st;
        }
        if ((st = bgk_step_boundary(c, stream)) != BGK_OK) return st;
    }
    return BGK_OK;
}

bgk_status bgk_buffer(bgk_ctx* c, bgk_buffer_id id, void** ptr, size_t* bytes) {
    if (!c || !ptr || !bytes) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, c->gstream);
    switch (id) {
        case BGK_BUF_MOMENT_SUMS: *ptr = c->sums; *bytes = sizeof(double) * c->N * kPM; return BGK_OK;
        case BGK_BUF_WALL_FLUX: *ptr = c->wallnum; *bytes = sizeof(double) * c->N; return BGK_OK;
        case BGK_BUF_F: *ptr = c->f[c->fcur]; *bytes = sizeof(double) * c->N * c->RS; return BGK_OK;
    }
    return BGK_E_INVALID_ARG;
}

bgk_status bgk_moments_partial(bgk_ctx* c, bgk_stream stream) {
    if (!c) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    launch_row_moments(c, c->f[c->fcur], S(stream));
    return check_launch(c);
}

bgk_status bgk_moments_finalize(bgk_ctx* c, double* rho, double* U, double* T, bgk_stream stream) {
    if (!c) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    cudaStream_t s = S(stream);
    launch_moments_finalize(c, c->outbuf, s);
    bgk_status st = check_launch(c);
    if (st == BGK_OK) st = sync_check(c, s);
    const int d = c->d;
    std::vector<double> h(c->N * (d + 2));
    cudaError_t e = cudaMemcpy(h.data(), c->outbuf, sizeof(double) * h.size(), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(c, e);
    std::vector<double> r(c->N), u(c->N * d), t(c->N);
    for (int64_t i = 0; i < c->N; ++i) {
        r[i] = h[i * (d + 2)];
        for (int a = 0; a < d; ++a) u[i * d + a] = h[i * (d + 2) + 1 + a];
        t[i] = h[i * (d + 2) + 1 + d];
    }
    if (rho) cudaMemcpy(rho, r.data(), sizeof(double) * c->N, cudaMemcpyDefault);
    if (U) cudaMemcpy(U, u.data(), sizeof(double) * c->N * d, cudaMemcpyDefault);
    if (T) cudaMemcpy(T, t.data(), sizeof(double) * c->N, cudaMemcpyDefault);
    return st;
}

bgk_status bgk_moments(bgk_ctx* c, double* rho, double* U, double* T, bgk_stream stream) {
    if (!c) return BGK_E_INVALID_ARG;
    if (c->ncol != c->ncol_g) return BGK_E_INVALID_ARG;
    bgk_status st = bgk_moments_partial(c, stream);
    if (st != BGK_OK) return st;
    return bgk_moments_finalize(c, rho, U, T, stream);
}

bgk_status bgk_get_macro(bgk_ctx* c, double* macro, bgk_stream stream) {
    if (!c || !macro) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    cudaStream_t s = S(stream);
    bgk_status st = copy_out(c, macro, c->macro, sizeof(double) * c->N * (c->d + 2), s);
    if (st != BGK_OK) return st;
    return sync_check(c, s);
}

bgk_status bgk_get_f(bgk_ctx* c, double* f, bgk_stream stream) {
    if (!c || !f) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    cudaStream_t s = S(stream);
    double* scratch = c->f[1 - c->fcur];
    launch_to_canonical(c, c->f[c->fcur], scratch, s);
    bgk_status st = check_launch(c);
    if (st != BGK_OK) return st;
    if ((st = copy_out(c, f, scratch, sizeof(double) * c->N * c->nv * c->Kloc, s)) != BGK_OK) return st;
    return sync_check(c, s);
}

bgk_status bgk_set_f(bgk_ctx* c, const double* f, bgk_stream stream) {
    if (!c || !f) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    cudaStream_t s = S(stream);
    double* scratch = c->f[1 - c->fcur];
    bgk_status st = copy_out(c, scratch, f, sizeof(double) * c->N * c->nv * c->Kloc, s);
    if (st != BGK_OK) return st;
    launch_from_canonical(c, scratch, c->f[c->fcur], s);
    if ((st = check_launch(c)) != BGK_OK) return st;
    return sync_check(c, s);
}

bgk_status bgk_get_positions(bgk_ctx* c, double* x, bgk_stream stream) {
    if (!c || !x) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    cudaStream_t s = S(stream);
    bgk_status st = copy_out(c, x, c->x, sizeof(double) * c->N * c->d, s);
    if (st != BGK_OK) return st;
    return sync_check(c, s);
}

bgk_status bgk_get_neighbors(bgk_ctx* c, int64_t* offsets, int32_t* idx, int64_t* nnz, bgk_stream stream) {
    if (!c) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    cudaStream_t s = S(stream);
    bgk_status st = sync_check(c, s);
    if (st != BGK_OK) return st;
    int64_t n = 0;
    cudaMemcpy(&n, c->g.nb_off + c->N, sizeof(int64_t), cudaMemcpyDeviceToHost);
    if (nnz) *nnz = n;
    if (offsets && (st = copy_out(c, offsets, c->g.nb_off, sizeof(int64_t) * (c->N + 1), s)) != BGK_OK) return st;
    if (idx && n && (st = copy_out(c, idx, c->g.nb_idx, sizeof(int32_t) * n, s)) != BGK_OK) return st;
    return sync_check(c, s);
}

bgk_status bgk_stable_dt(bgk_ctx* c, double* dt_out, bgk_stream stream) {
    if (!c || !dt_out) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    cudaStream_t s = S(stream);
    bgk_status st0 = ensure_geometry(c, s);
    if (st0 != BGK_OK) return st0;
    cudaMemsetAsync(c->stab, 0, sizeof(unsigned long long), s);
    launch_transport(c, c->f[c->fcur], c->f[1 - c->fcur], s);
    bgk_status st = check_launch(c);
    if (st == BGK_OK) st = sync_check(c, s);
    if (st != BGK_OK) return st;
    unsigned long long bits = 0;
    cudaMemcpy(&bits, c->stab, sizeof(bits), cudaMemcpyDeviceToHost);
    double m;
    std::memcpy(&m, &bits, sizeof(m));
    *dt_out = m > 0.0 ? 1.0 / m : INFINITY;
    return BGK_OK;
}

bgk_status bgk_launches_per_step(bgk_ctx* c, int64_t* n) {
    if (!c || !n) return BGK_E_INVALID_ARG;
    int64_t k = 0;
    if (c->cfg.ale) k += launches_neighbors(c) + launches_wls() - (c->N_b ? 0 : 1) - (c->N_int ? 0 : 1);
    if (c->cfg.ale && c->N_b) k += 1;   // k_bnd_union
    if (c->cfg.ale && c->cfg.manage)   // k_mg_detect_w (+ k_mg_detect_wall) + k_mg_decide (plus 3 more and a
        k += 2 + (c->N_b ? 1 : 0);     // neighbour rebuild in the rare steps where the cloud changes)
    if (c->cfg.ale && c->cfg.manage && c->graph_ok && c->ncol == c->ncol_g)
        k += 3;                  // graph steps: the two conditional gates and the step counter (graph.cu)
    if (c->N_int) k += c->fuse2 ? 1 : 3 + (c->fold ? 1 : 0);   // transport (+ the folded group), moment
                                                                 // reduce, relax -- or the fused kernel
    if (c->rows_built) k += (c->n_tiles > 0) + (c->n_rows > 0) - (c->n_rest == 0);   // fixed cloud
    if (c->N_b) k += 3;          // boundary interp, wall reduce, fill
    *n = k;
    return BGK_OK;
}

bgk_status bgk_sync(bgk_ctx* c, bgk_stream stream) {
    if (!c) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    return sync_check(c, S(stream));
}

const char* bgk_last_error(bgk_ctx* c, int64_t* particle) {
    if (!c) return "null context";
    if (particle) *particle = c->bad;
    return c->msg;
}

bgk_status bgk_destroy(bgk_ctx* c) {
    if (c) graph_release(c);
    if (c && c->cfg.staging) {
        cudaEventDestroy(c->ev_staged);
        cudaEventDestroy(c->ev_consumed);
    }
    delete c;
    return BGK_OK;
}

bgk_status bgk_stage_f(bgk_ctx* c, const double* f, bgk_stream copy_stream) {
    if (!c || !f || !c->cfg.staging) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, c->gstream);
    cudaStream_t cs = S(copy_stream);
    cudaError_t e = cudaStreamWaitEvent(cs, c->ev_consumed, 0);   // the previous staged input is converted
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(c->stage, f, sizeof(double) * c->N * c->nv * c->Kloc, cudaMemcpyDefault, cs);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_staged, cs);
    if (e != cudaSuccess) return cuda_fail(c, e);
    c->stage_pending = true;
    c->stage_N = c->N;                 // the staged rows belong to this cloud (size and numbering)
    c->stage_gen = c->cloud_gen;
    return BGK_OK;
}

bgk_status bgk_use_staged_f(bgk_ctx* c, bgk_stream stream) {
    if (!c || !c->cfg.staging || !c->stage_pending) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    if (c->stage_N != c->N || c->stage_gen != c->cloud_gen) {
        // particle management changed N or renumbered the rows after bgk_stage_f: the staged
        // rows no longer match the cloud (the copy itself completed within the old size)
        std::snprintf(c->msg, sizeof(c->msg), "staged f was copied for %lld particles before the cloud changed "
                      "(now %lld); stage it again", (long long)c->stage_N, (long long)c->N);
        c->bad = -1;
        c->stage_pending = false;
        return BGK_E_INVALID_ARG;
    }
    cudaStream_t s = S(stream);
    cudaError_t e = cudaStreamWaitEvent(s, c->ev_staged, 0);
    if (e != cudaSuccess) return cuda_fail(c, e);
    launch_from_canonical(c, c->stage, c->f[c->fcur], s);
    e = cudaEventRecord(c->ev_consumed, s);
    if (e != cudaSuccess) return cuda_fail(c, e);
    c->stage_pending = false;
    return check_launch(c);
}

bgk_status bgk_manage(bgk_ctx* c, int64_t* report, bgk_stream stream) {
    if (!c) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    if (!c->cfg.manage) return BGK_E_INVALID_ARG;   // no scratch carved
    cudaStream_t s = S(stream);
    launch_build_neighbors(c, s);
    bool changed = false;
    bgk_status st = manage_pass(c, s, &changed);
    c->geometry_valid = false;
    if (st == BGK_OK) st = sync_check(c, s);
    if (report) std::memcpy(report, c->mg_report, sizeof(c->mg_report));
    return st;
}

bgk_status bgk_count(bgk_ctx* c, int64_t* N, int64_t* n_interior, int64_t* n_boundary, int64_t* capacity) {
    if (!c) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, c->gstream);
    if (N) *N = c->N;
    if (n_interior) *n_interior = c->N_int;
    if (n_boundary) *n_boundary = c->N_b;
    if (capacity) *capacity = c->Ncap;
    return BGK_OK;
}

bgk_status bgk_transport_info(bgk_ctx* c, int64_t* info) {
    if (!c || !info) return BGK_E_INVALID_ARG;
    info[0] = 1;                      // particles per transport warp
    info[1] = c->R;
    info[2] = c->rows_built ? c->n_rows : 0;
    info[3] = c->rows_built ? c->n_rest : c->N_int;
    info[4] = c->rows_built ? c->n_tiles : 0;
    return BGK_OK;
}

bgk_status bgk_manage_report(bgk_ctx* c, int64_t* report) {
    if (!c || !report) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, c->gstream);
    std::memcpy(report, c->mg_report, sizeof(c->mg_report));
    return BGK_OK;
}

bgk_status bgk_get_kind(bgk_ctx* c, int8_t* kind, bgk_stream stream) {
    if (!c || !kind) return BGK_E_INVALID_ARG;
    BGK_RECONCILE(c, S(stream));
    cudaStream_t s = S(stream);
    bgk_status st = copy_out(c, kind, c->kind, (size_t)c->N, s);
    if (st != BGK_OK) return st;
    return sync_check(c, s);
}

}  // extern "C"
