// cc_band.h — the device-resident row-band iteration (BASELINE config 5,
// SURVEY.md §8e): the exchange between band trainers runs on their streams,
// so a run of proxy iterations (encoder.hpp:97-135) is enqueued without any
// host synchronisation.  Per iteration, on every band b:
//
//   A  latent halo rows y: owner -> neighbours
//   B  forward + backward on the band (Trainer::band_dev_forward_backward)
//   C  partial latent gradients of halo rows: neighbour -> owner, added
//      (from the band above first, then from the band below)
//   D  [NN-gradient partials | bits | squared error] gathered from all bands
//   E  rank-order fp64 sums -> gradients, per-tensor flags, the global cost;
//      own-row latent-gradient finiteness per grid
//   F  per-grid flags AND-ed over the bands
//   G  latent + NN Adam (identical on every band), the iteration's record
//
// Two transports share that sequence and the row routing:
//   * local: every band of the image in this process (one GPU or several):
//     device-to-device / peer copies ordered by events between the streams;
//   * NCCL: one band per process; grouped ncclSend/ncclRecv for A and C,
//     ncclAllGather for D, ncclAllReduce(min) for F, all on the band's stream
//     (libnccl.so.2 is resolved at run time — the one torch.distributed
//     already loaded).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "cc_runtime.h"

namespace ccb {

// global grid rows of one band at one level: window [w0, w1) ⊇ own [o0, o1)
struct BandRows {
    int w0, o0, o1, w1;
};
BandRows band_rows_at(int hg, int r0, int r1, int halo, int level, int grows);

// per grid, the global row ranges band b exchanges (bands.py halo_plan)
struct BandLink {
    int cols = 0;
    int send_up[2] = {0, 0}, send_down[2] = {0, 0};  // own rows neighbour b-1 / b+1 holds as halo
    int halo_up[2] = {0, 0}, halo_down[2] = {0, 0};  // window rows owned by b-1 / b+1
};
std::vector<BandLink> band_links(const Trainer& tr, const int* edges, int nbands, int b);

struct NcclComm;

// returned halo gradients: latent-gradient element offset, staging offset, count
struct BandSeg {
    int64_t dst, src, n;
};

class BandGroup {
public:
    explicit BandGroup(std::vector<Trainer*> bands);  // local transport
    BandGroup(Trainer* band, const void* nccl_id, int nranks, int rank, const int* edges);  // NCCL
    ~BandGroup();
    BandGroup(const BandGroup&) = delete;
    BandGroup& operator=(const BandGroup&) = delete;

    void reserve(int n);
    void enqueue_proxy_iterations(int n, const double* lr, const double* temp, const double* noise);
    void synchronize();
    static void nccl_unique_id(void* out128);

private:
    using Seg = BandSeg;
    struct Side {
        Trainer* tr = nullptr;
        int rank = 0;
        std::vector<BandLink> links;
        double* pack = nullptr;      // [n_params + 2]
        double* gathered = nullptr;  // [nbands][n_params + 2]
        float* stage = nullptr;      // returned halo gradients: [up segments | down segments]
        int* okpub = nullptr;        // local transport: this band's flags, published
        int* okall = nullptr;        // local transport: [nbands][kMaxGrids]
        Seg* d_up = nullptr;
        Seg* d_down = nullptr;
        int n_up = 0, n_down = 0;
        int64_t stage_up = 0, stage_down = 0;  // elements
        cudaEvent_t ev = nullptr;
    };
    void setup(Side& s, const int* edges);
    void iteration();
    void barrier();
    void halo_rows_local(int b);
    void grads_back_local(int b);
    void iteration_nccl();
    float* rows(Side& s, int which, int gi, const int* r);

    std::vector<Side> sides_;
    int nbands_ = 0;
    int64_t pack_n_ = 0;
    NcclComm* nccl_ = nullptr;
};

}  // namespace ccb
