// cc_band.cu — device-resident row-band iteration: the exchange kernels, the
// local (in-process) and NCCL transports.  See cc_band.h for the phase list;
// the host-driven version of the same iteration is bands.py (LocalBands /
// DistBand) over include/coolchic_b200_band.h, and both give bit-identical
// states (tests/test_bands.py).
#include "cc_band.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <type_traits>

namespace ccb {

namespace {

// E: rank-order fp64 sums of the gathered partials (every band adds the same
// values in the same order, so all bands hold bit-identical gradients), the
// per-tensor finiteness flags of adam_step (optim.hpp:38-41) and the global
// cost (encoder.hpp:111-118).  One CTA per NN tensor.
__global__ void __launch_bounds__(256) k_band_finish(const Plan* __restrict__ pp, const double* __restrict__ parts,
                                                     int nparts, int64_t stride) {
    const Plan& P = *pp;
    const int ti = blockIdx.x;
    const int off = P.tensor_off[ti], n = P.tensor_size[ti];
    int bad = 0;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int p = off + e;
        double s = 0.0;
        for (int r = 0; r < nparts; ++r) s += parts[r * stride + p];
        const float g = float(s);
        P.grads[p] = g;
        bad |= isfinite(g) ? 0 : 1;
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) P.tensor_ok[ti] = bad ? 0 : 1;
    if (ti == 0 && threadIdx.x == 0) {
        double bits = 0.0, se = 0.0;
        for (int r = 0; r < nparts; ++r) {
            bits += parts[r * stride + P.n_params];
            se += parts[r * stride + P.n_params + 1];
        }
        const double mse = se / double(3 * P.npix_global);
        // encoder.hpp:115, contracted as the reference build (-ffp-contract=fast) and k_finalize do
        const double cost = fma(P.lambda, bits / double(P.npix_global), mse);
        DevScalars* s = P.scal;
        s->bits = bits;
        s->mse = mse;
        s->cost = cost;
        s->cost_ok = isfinite(cost) ? 1 : 0;
        s->halt = 0;  // bands: the global cost decides
    }
}

// D: this band's [NN-gradient partials | bits | squared error]
__global__ void k_band_pack(const Plan* __restrict__ pp, double* __restrict__ dst) {
    const Plan& P = *pp;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P.n_params; p += gridDim.x * blockDim.x)
        dst[p] = P.grads_d[p];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        dst[P.n_params] = P.scal->bits;
        dst[P.n_params + 1] = P.scal->mse * double(3 * P.npix_global);
    }
}

// C: returned halo gradients added onto the owner's rows, one segment per y-block
__global__ void k_band_add(float* __restrict__ lat_g, const float* __restrict__ stage,
                           const BandSeg* __restrict__ segs) {
    const BandSeg sg = segs[blockIdx.y];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < sg.n; i += int64_t(gridDim.x) * blockDim.x)
        lat_g[sg.dst + i] += stage[sg.src + i];
}

// F (local transport): AND over the bands' per-grid flags
__global__ void k_band_ok_min(int* __restrict__ lat_ok, const int* __restrict__ all, int nparts, int ngrids) {
    const int g = threadIdx.x;
    if (g >= ngrids) return;
    int v = 1;
    for (int r = 0; r < nparts; ++r) v = min(v, all[r * kMaxGrids + g]);
    lat_ok[g] = v;
}

void copy_dev(void* dst, int ddev, const void* src, int sdev, size_t bytes, cudaStream_t st) {
    if (!bytes) return;
    if (ddev == sdev)
        CCB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
    else
        CCB_CUDA(cudaMemcpyPeerAsync(dst, ddev, src, sdev, bytes, st));
}

}  // namespace

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclComm {
    ncclComm_t comm = nullptr;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;

    static NcclComm* load() {
        // the library torch.distributed loaded (same soname), else the search path
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) throw ConfigError(std::string("NCCL transport: cannot load libnccl.so.2: ") + dlerror());
        auto* n = new NcclComm();
        auto sym = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp) {
                delete n;
                throw ConfigError(std::string("NCCL transport: missing symbol ") + name);
            }
        };
        sym(n->getUniqueId, "ncclGetUniqueId");
        sym(n->commInitRank, "ncclCommInitRank");
        sym(n->commDestroy, "ncclCommDestroy");
        sym(n->groupStart, "ncclGroupStart");
        sym(n->groupEnd, "ncclGroupEnd");
        sym(n->send, "ncclSend");
        sym(n->recv, "ncclRecv");
        sym(n->allGather, "ncclAllGather");
        sym(n->allReduce, "ncclAllReduce");
        sym(n->errorString, "ncclGetErrorString");
        return n;
    }
    void check(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess && r != ncclInProgress)
            throw CudaError(std::string(what) + ": " + (errorString ? errorString(r) : "nccl error"));
    }
};

// ---------------------------------------------------------------- row routing
BandRows band_rows_at(int hg, int r0, int r1, int halo, int level, int grows) {
    // Trainer::build_plan's band geometry (cc_runtime.cu), bands.py band_grid_rows
    const int o0 = r0 >> level;
    const int o1 = r1 == hg ? grows : r1 >> level;
    return {std::max(0, o0 - halo), o0, o1, std::min(grows, o1 + halo)};
}

std::vector<BandLink> band_links(const Trainer& tr, const int* edges, int nbands, int b) {
    int hg, r0, r1, halo;
    tr.band_spec(&hg, &r0, &r1, &halo);
    if (edges[b] != r0 || edges[b + 1] != r1) throw ConfigError("band rows do not match the band edges");
    if (edges[0] != 0 || edges[nbands] != hg) throw ConfigError("band edges do not cover the image");
    const Plan& H = tr.host_plan();
    std::vector<BandLink> out(size_t(H.n_grids));
    for (int gi = 0; gi < H.n_grids; ++gi) {
        const GridGeom& g = H.g[gi];
        const BandRows me = band_rows_at(hg, r0, r1, halo, g.level, g.grows);
        if (me.w0 != g.row0 || me.o0 != g.row0 + g.own_lo || me.o1 != g.row0 + g.own_hi || me.w1 != g.row0 + g.rows)
            throw ConfigError("band geometry mismatch");
        BandLink& L = out[size_t(gi)];
        L.cols = g.cols;
        L.halo_up[0] = me.w0, L.halo_up[1] = me.o0;
        L.halo_down[0] = me.o1, L.halo_down[1] = me.w1;
        if (b > 0) {
            const BandRows up = band_rows_at(hg, edges[b - 1], edges[b], halo, g.level, g.grows);
            if (up.o0 > me.w0) throw ConfigError("halo deeper than the neighbouring band");
            L.send_up[0] = me.o0, L.send_up[1] = up.w1;
        }
        if (b + 1 < nbands) {
            const BandRows dn = band_rows_at(hg, edges[b + 1], edges[b + 2], halo, g.level, g.grows);
            if (dn.o1 < me.w1) throw ConfigError("halo deeper than the neighbouring band");
            L.send_down[0] = dn.w0, L.send_down[1] = me.o1;
        }
    }
    return out;
}

// ---------------------------------------------------------------- group
float* BandGroup::rows(Side& s, int which, int gi, const int* r) {
    int64_t n = 0;
    return static_cast<float*>(s.tr->band_device_rows(which, gi, r[0], r[1], &n));
}

void BandGroup::setup(Side& s, const int* edges) {
    Trainer& tr = *s.tr;
    const Plan& H = tr.host_plan();
    CCB_CUDA(cudaSetDevice(tr.device()));
    s.links = band_links(tr, edges, nbands_, s.rank);
    pack_n_ = H.n_params + 2;
    CCB_CUDA(cudaMalloc(&s.pack, sizeof(double) * size_t(pack_n_)));
    CCB_CUDA(cudaMalloc(&s.gathered, sizeof(double) * size_t(pack_n_) * size_t(nbands_)));
    CCB_CUDA(cudaMalloc(&s.okpub, sizeof(int) * kMaxGrids));
    CCB_CUDA(cudaMalloc(&s.okall, sizeof(int) * kMaxGrids * size_t(nbands_)));
    CCB_CUDA(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
    // staging of returned halo gradients: rows send_up (from b-1), then send_down (from b+1)
    std::vector<Seg> up, dn;
    int64_t pos = 0;
    for (int gi = 0; gi < H.n_grids; ++gi) {
        const BandLink& L = s.links[size_t(gi)];
        const GridGeom& g = H.g[gi];
        const int64_t n = int64_t(L.send_up[1] - L.send_up[0]) * L.cols;
        if (n > 0) up.push_back({g.lat_off + int64_t(L.send_up[0] - g.row0) * g.cols, pos, n}), pos += n;
    }
    s.stage_up = pos;
    for (int gi = 0; gi < H.n_grids; ++gi) {
        const BandLink& L = s.links[size_t(gi)];
        const GridGeom& g = H.g[gi];
        const int64_t n = int64_t(L.send_down[1] - L.send_down[0]) * L.cols;
        if (n > 0) dn.push_back({g.lat_off + int64_t(L.send_down[0] - g.row0) * g.cols, pos, n}), pos += n;
    }
    s.stage_down = pos - s.stage_up;
    s.n_up = int(up.size()), s.n_down = int(dn.size());
    CCB_CUDA(cudaMalloc(&s.stage, sizeof(float) * size_t(std::max<int64_t>(pos, 1))));
    if (!up.empty()) {
        CCB_CUDA(cudaMalloc(&s.d_up, sizeof(Seg) * up.size()));
        CCB_CUDA(cudaMemcpy(s.d_up, up.data(), sizeof(Seg) * up.size(), cudaMemcpyHostToDevice));
    }
    if (!dn.empty()) {
        CCB_CUDA(cudaMalloc(&s.d_down, sizeof(Seg) * dn.size()));
        CCB_CUDA(cudaMemcpy(s.d_down, dn.data(), sizeof(Seg) * dn.size(), cudaMemcpyHostToDevice));
    }
}

BandGroup::BandGroup(std::vector<Trainer*> bands) {
    if (bands.empty()) throw ConfigError("a band group needs at least one band");
    nbands_ = int(bands.size());
    std::vector<int> edges(size_t(nbands_) + 1);
    for (int b = 0; b < nbands_; ++b) {
        if (!bands[size_t(b)] || !bands[size_t(b)]->is_band()) throw ConfigError("not a band trainer");
        int hg, r0, r1, halo;
        bands[size_t(b)]->band_spec(&hg, &r0, &r1, &halo);
        if (b > 0 && edges[size_t(b)] != r0) throw ConfigError("bands must be contiguous and in row order");
        edges[size_t(b)] = r0;
        edges[size_t(b) + 1] = r1;
        if (bands[size_t(b)]->host_plan().n_params != bands[0]->host_plan().n_params)
            throw ConfigError("bands of one image must share the decoder");
    }
    sides_.resize(size_t(nbands_));
    for (int b = 0; b < nbands_; ++b) {
        sides_[size_t(b)].tr = bands[size_t(b)];
        sides_[size_t(b)].rank = b;
        setup(sides_[size_t(b)], edges.data());
    }
}

BandGroup::BandGroup(Trainer* band, const void* nccl_id, int nranks, int rank, const int* edges) {
    if (!band || !band->is_band()) throw ConfigError("not a band trainer");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw ConfigError("bad NCCL rank / size");
    nbands_ = nranks;
    sides_.resize(1);
    sides_[0].tr = band;
    sides_[0].rank = rank;
    setup(sides_[0], edges);
    nccl_ = NcclComm::load();
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    CCB_CUDA(cudaSetDevice(band->device()));
    nccl_->check(nccl_->commInitRank(&nccl_->comm, nranks, id, rank), "ncclCommInitRank");
}

void BandGroup::nccl_unique_id(void* out128) {
    NcclComm* n = NcclComm::load();
    ncclUniqueId id;
    const ncclResult_t r = n->getUniqueId(&id);
    const std::string msg = r == ncclSuccess ? "" : n->errorString(r);
    delete n;
    if (r != ncclSuccess) throw CudaError("ncclGetUniqueId: " + msg);
    std::memcpy(out128, &id, sizeof(id));
}

BandGroup::~BandGroup() {
    for (Side& s : sides_) {
        cudaSetDevice(s.tr->device());
        cudaStreamSynchronize(s.tr->stream());
        cudaFree(s.pack);
        cudaFree(s.gathered);
        cudaFree(s.stage);
        cudaFree(s.okpub);
        cudaFree(s.okall);
        cudaFree(s.d_up);
        cudaFree(s.d_down);
        if (s.ev) cudaEventDestroy(s.ev);
    }
    if (nccl_) {
        if (nccl_->comm) nccl_->commDestroy(nccl_->comm);
        delete nccl_;
    }
}

void BandGroup::reserve(int n) {
    for (Side& s : sides_) s.tr->band_reserve(n);
}

// every band's stream waits for every other band's work enqueued so far
void BandGroup::barrier() {
    if (sides_.size() < 2) return;
    for (Side& s : sides_) {
        CCB_CUDA(cudaSetDevice(s.tr->device()));
        CCB_CUDA(cudaEventRecord(s.ev, s.tr->stream()));
    }
    for (Side& s : sides_) {
        CCB_CUDA(cudaSetDevice(s.tr->device()));
        for (Side& o : sides_)
            if (&o != &s) CCB_CUDA(cudaStreamWaitEvent(s.tr->stream(), o.ev, 0));
    }
}

// A (local): band b pulls its halo latents from the owners
void BandGroup::halo_rows_local(int b) {
    Side& s = sides_[size_t(b)];
    const int dev = s.tr->device();
    cudaStream_t st = s.tr->stream();
    for (size_t gi = 0; gi < s.links.size(); ++gi) {
        const BandLink& L = s.links[gi];
        if (b > 0 && L.halo_up[1] > L.halo_up[0]) {
            Side& o = sides_[size_t(b) - 1];
            copy_dev(rows(s, 0, int(gi), L.halo_up), dev, rows(o, 0, int(gi), L.halo_up), o.tr->device(),
                     sizeof(float) * size_t(L.halo_up[1] - L.halo_up[0]) * size_t(L.cols), st);
        }
        if (b + 1 < nbands_ && L.halo_down[1] > L.halo_down[0]) {
            Side& o = sides_[size_t(b) + 1];
            copy_dev(rows(s, 0, int(gi), L.halo_down), dev, rows(o, 0, int(gi), L.halo_down), o.tr->device(),
                     sizeof(float) * size_t(L.halo_down[1] - L.halo_down[0]) * size_t(L.cols), st);
        }
    }
}

// C (local): band b pulls the gradients its neighbours computed for b's own rows
void BandGroup::grads_back_local(int b) {
    Side& s = sides_[size_t(b)];
    const int dev = s.tr->device();
    cudaStream_t st = s.tr->stream();
    int64_t pos = 0;
    for (size_t gi = 0; gi < s.links.size() && b > 0; ++gi) {
        const BandLink& L = s.links[gi];
        const int64_t n = int64_t(L.send_up[1] - L.send_up[0]) * L.cols;
        if (n <= 0) continue;
        Side& o = sides_[size_t(b) - 1];
        copy_dev(s.stage + pos, dev, rows(o, 1, int(gi), L.send_up), o.tr->device(), sizeof(float) * size_t(n), st);
        pos += n;
    }
    for (size_t gi = 0; gi < s.links.size() && b + 1 < nbands_; ++gi) {
        const BandLink& L = s.links[gi];
        const int64_t n = int64_t(L.send_down[1] - L.send_down[0]) * L.cols;
        if (n <= 0) continue;
        Side& o = sides_[size_t(b) + 1];
        copy_dev(s.stage + pos, dev, rows(o, 1, int(gi), L.send_down), o.tr->device(), sizeof(float) * size_t(n), st);
        pos += n;
    }
}

void BandGroup::iteration() {
    if (nccl_) return iteration_nccl();
    const int B = nbands_;
    barrier();  // the owners' latents of the last step are final
    for (int b = 0; b < B; ++b) {
        CCB_CUDA(cudaSetDevice(sides_[size_t(b)].tr->device()));
        halo_rows_local(b);
        sides_[size_t(b)].tr->band_dev_forward_backward();
    }
    barrier();  // every band's latent gradients are complete
    for (int b = 0; b < B; ++b) {
        Side& s = sides_[size_t(b)];
        CCB_CUDA(cudaSetDevice(s.tr->device()));
        grads_back_local(b);
        const Plan& H = s.tr->host_plan();
        if (s.n_up)
            k_band_add<<<dim3(32, s.n_up), 256, 0, s.tr->stream()>>>(H.lat_g, s.stage, s.d_up);
        if (s.n_down)
            k_band_add<<<dim3(32, s.n_down), 256, 0, s.tr->stream()>>>(H.lat_g, s.stage, s.d_down);
        k_band_pack<<<8, 256, 0, s.tr->stream()>>>(s.tr->device_plan(), s.pack);
    }
    barrier();  // every band's partials are packed
    for (int b = 0; b < B; ++b) {
        Side& s = sides_[size_t(b)];
        CCB_CUDA(cudaSetDevice(s.tr->device()));
        for (int k = 0; k < B; ++k)
            copy_dev(s.gathered + size_t(k) * size_t(pack_n_), s.tr->device(), sides_[size_t(k)].pack,
                     sides_[size_t(k)].tr->device(), sizeof(double) * size_t(pack_n_), s.tr->stream());
        const Plan& H = s.tr->host_plan();
        k_band_finish<<<H.n_tensors, 256, 0, s.tr->stream()>>>(s.tr->device_plan(), s.gathered, B, pack_n_);
        launch_band_own_finite(s.tr->launch_ctx());
        CCB_CUDA(cudaMemcpyAsync(s.okpub, H.lat_ok, sizeof(int) * kMaxGrids, cudaMemcpyDeviceToDevice,
                                 s.tr->stream()));
    }
    barrier();  // every band's flags are published
    for (int b = 0; b < B; ++b) {
        Side& s = sides_[size_t(b)];
        CCB_CUDA(cudaSetDevice(s.tr->device()));
        for (int k = 0; k < B; ++k)
            copy_dev(s.okall + size_t(k) * kMaxGrids, s.tr->device(), sides_[size_t(k)].okpub,
                     sides_[size_t(k)].tr->device(), sizeof(int) * kMaxGrids, s.tr->stream());
        const Plan& H = s.tr->host_plan();
        k_band_ok_min<<<1, 32, 0, s.tr->stream()>>>(H.lat_ok, s.okall, B, H.n_grids);
        s.tr->band_dev_step();
    }
}

void BandGroup::iteration_nccl() {
    Side& s = sides_[0];
    Trainer& tr = *s.tr;
    const Plan& H = tr.host_plan();
    const int r = s.rank;
    cudaStream_t st = tr.stream();
    const NcclComm& N = *nccl_;
    CCB_CUDA(cudaSetDevice(tr.device()));
    // A: y rows, one message per grid and direction (matched in grid order)
    N.check(N.groupStart(), "ncclGroupStart");
    for (size_t gi = 0; gi < s.links.size(); ++gi) {
        const BandLink& L = s.links[gi];
        if (r > 0) {
            const size_t ns = size_t(L.send_up[1] - L.send_up[0]) * size_t(L.cols);
            const size_t nr = size_t(L.halo_up[1] - L.halo_up[0]) * size_t(L.cols);
            if (ns) N.check(N.send(rows(s, 0, int(gi), L.send_up), ns, ncclFloat32, r - 1, N.comm, st), "ncclSend");
            if (nr) N.check(N.recv(rows(s, 0, int(gi), L.halo_up), nr, ncclFloat32, r - 1, N.comm, st), "ncclRecv");
        }
        if (r + 1 < nbands_) {
            const size_t ns = size_t(L.send_down[1] - L.send_down[0]) * size_t(L.cols);
            const size_t nr = size_t(L.halo_down[1] - L.halo_down[0]) * size_t(L.cols);
            if (ns) N.check(N.send(rows(s, 0, int(gi), L.send_down), ns, ncclFloat32, r + 1, N.comm, st), "ncclSend");
            if (nr) N.check(N.recv(rows(s, 0, int(gi), L.halo_down), nr, ncclFloat32, r + 1, N.comm, st), "ncclRecv");
        }
    }
    N.check(N.groupEnd(), "ncclGroupEnd");
    // B
    tr.band_dev_forward_backward();
    // C: halo-row gradients to the owners; own rows' gradients from the neighbours
    N.check(N.groupStart(), "ncclGroupStart");
    int64_t pos_up = 0, pos_dn = s.stage_up;
    for (size_t gi = 0; gi < s.links.size(); ++gi) {
        const BandLink& L = s.links[gi];
        if (r > 0) {
            const size_t ns = size_t(L.halo_up[1] - L.halo_up[0]) * size_t(L.cols);
            const size_t nr = size_t(L.send_up[1] - L.send_up[0]) * size_t(L.cols);
            if (ns) N.check(N.send(rows(s, 1, int(gi), L.halo_up), ns, ncclFloat32, r - 1, N.comm, st), "ncclSend");
            if (nr) N.check(N.recv(s.stage + pos_up, nr, ncclFloat32, r - 1, N.comm, st), "ncclRecv");
            pos_up += int64_t(nr);
        }
        if (r + 1 < nbands_) {
            const size_t ns = size_t(L.halo_down[1] - L.halo_down[0]) * size_t(L.cols);
            const size_t nr = size_t(L.send_down[1] - L.send_down[0]) * size_t(L.cols);
            if (ns) N.check(N.send(rows(s, 1, int(gi), L.halo_down), ns, ncclFloat32, r + 1, N.comm, st), "ncclSend");
            if (nr) N.check(N.recv(s.stage + pos_dn, nr, ncclFloat32, r + 1, N.comm, st), "ncclRecv");
            pos_dn += int64_t(nr);
        }
    }
    N.check(N.groupEnd(), "ncclGroupEnd");
    if (s.n_up) k_band_add<<<dim3(32, s.n_up), 256, 0, st>>>(H.lat_g, s.stage, s.d_up);
    if (s.n_down) k_band_add<<<dim3(32, s.n_down), 256, 0, st>>>(H.lat_g, s.stage, s.d_down);
    // D, E
    k_band_pack<<<8, 256, 0, st>>>(tr.device_plan(), s.pack);
    N.check(N.allGather(s.pack, s.gathered, size_t(pack_n_), ncclFloat64, N.comm, st), "ncclAllGather");
    k_band_finish<<<H.n_tensors, 256, 0, st>>>(tr.device_plan(), s.gathered, nbands_, pack_n_);
    launch_band_own_finite(tr.launch_ctx());
    // F, G
    N.check(N.allReduce(H.lat_ok, H.lat_ok, size_t(H.n_grids), ncclInt32, ncclMin, N.comm, st), "ncclAllReduce");
    tr.band_dev_step();
}

void BandGroup::enqueue_proxy_iterations(int n, const double* lr, const double* temp, const double* noise) {
    if (n <= 0) return;
    reserve(n);
    for (Side& s : sides_) {
        CCB_CUDA(cudaSetDevice(s.tr->device()));
        s.tr->upload_schedule(n, lr, temp, noise);
        s.tr->reset_batch_counters();
    }
    for (int i = 0; i < n; ++i) iteration();
    CCB_CUDA(cudaGetLastError());
}

void BandGroup::synchronize() {
    for (Side& s : sides_) s.tr->synchronize();
}

}  // namespace ccb
