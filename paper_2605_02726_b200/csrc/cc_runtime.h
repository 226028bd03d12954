// cc_runtime.h — host side of the B200 trainer: geometry, device arena, the
// per-iteration launch sequences (captured once as CUDA graphs), and the
// reference's Trainer surface (encoder.hpp:59-306) on top of them.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/coolchic_b200.h"
#include "cc_kernels.h"
#include "cc_plan.h"

namespace ccb {

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what);
#define CCB_CUDA(x) ::ccb::cuda_check((x), #x)

struct TensorInfo {
    std::string name;
    int rows, cols;
    int size, offset;
};

struct GridInfo {
    int level, hyper, rows, cols;
    int64_t offset;
    int ifce_slot;
};

// Device buffers of one CandidateState (encoder.hpp:42-48).
struct CandSlot {
    float *y = nullptr, *m = nullptr, *v = nullptr, *p = nullptr, *nm = nullptr, *nv = nullptr;
    double* soap = nullptr;
    std::vector<int64_t> lat_t, nn_t;
    double cost = 0.0;
};

struct SnapSlot {
    float *y = nullptr, *p = nullptr;
    bool valid = false;
};

class Trainer {
public:
    Trainer(const float* image, int h, int w, const cc_encoder_config& enc,
            const cc_decoder_config& dec, int device);
    // one row band [r0, r1) of an hg x w image (cfg5); image_window holds the
    // pixel rows band_window() returns
    Trainer(const float* image_window, int hg, int w, int r0, int r1, int halo,
            const cc_encoder_config& enc, const cc_decoder_config& dec, int device);
    static void band_window(int hg, int w, int r0, int r1, int halo, int* w0, int* w1);
    ~Trainer();
    Trainer(const Trainer&) = delete;
    Trainer& operator=(const Trainer&) = delete;

    // ---- reference surface ----
    void upload_image(const float* image);
    void fresh_candidate(int index);
    double proxy_iteration(double lr, double temp, double noise_std);
    // n iterations without host round trips; rec receives 4 doubles per
    // iteration (cost, mse, bits, global_iter after the iteration)
    void proxy_iterations(int n, const double* lr, const double* temp, const double* noise,
                          double* rec);
    void enqueue_proxy_iterations(int n, const double* lr, const double* temp, const double* noise);
    // size the batch buffers for n iterations and instantiate the batched graph
    // (one-off setup kept out of enqueue_proxy_iterations' steady state)
    void reserve_iterations(int n);
    void last_records(int n, double* rec);
    // batched images (cfg3): capture this trainer's proxy iteration as ONE graph
    // of launches over `batch` consecutive device plans (every kernel reads
    // pp[blockIdx.z]); the plans must share this trainer's geometry.
    cudaGraphExec_t capture_batched_proxy(const Plan* d_plans, int batch, float* const* arm_cstages);
    void upload_schedule(int n, const double* lr, const double* temp, const double* noise);
    void reset_batch_counters();
    const Plan& host_plan() const { return H_; }
    const double* device_schedule() const { return d_sched_; }
    cudaStream_t stream() const { return stream_; }
    void set_stream(cudaStream_t s);
    void profile_stages(int n, double lr, double temp, double noise, double* ms);
    static constexpr int kTimelineMarks = 13;
    void timeline(int n, double lr, double temp, double noise, double* ms);
    int kernels_per_iteration();
    double hardround_iteration(double lr, int best_slot);
    double true_cost(double* psnr, double* bpp);
    void quantize_all();
    void load_pads_from_q();
    void snapshot(int slot, double cost);
    double snapshot_cost(int slot);
    void restore(int slot);
    void reset_optimizers();
    void take_candidate(int slot, double cost);
    void load_candidate(int slot);
    void discard_candidate(int slot);
    double candidate_cost(int slot) const;
    double last_mse() const { return last_mse_; }
    double last_bits() const { return last_bits_; }
    int64_t global_iter();
    int skipped_steps();
    void set_counters(int64_t gi, int skipped);
    double current_cost() const { return cur_cost_; }
    void set_current_cost(double c) { cur_cost_ = c; }

    // row bands (cfg5): see cc_runtime.cu
    bool is_band() const { return band_.on; }
    void band_spec(int* hg, int* r0, int* r1, int* halo) const {
        *hg = band_.hg, *r0 = band_.r0, *r1 = band_.r1, *halo = band_.halo;
    }
    void band_forward_backward(double lr, double temp, double noise, double* bits, double* se);
    void band_nn_partial(double* out);
    double band_finish(const double* nn_sums, double bits, double se, int* lat_ok_own);
    void band_step(const int* lat_ok);
    void band_rows(int which, int gi, int rb, int re, float* buf, int mode);
    void band_grid_rows(int gi, int* out4) const;
    void* band_device_rows(int which, int gi, int rb, int re, int64_t* count);
    double* nn_partial_device() { return H_.grads_d; }
    // device-resident band iteration (cc_band.cu drives the exchange between
    // the phases; no host synchronisation inside an iteration)
    void band_reserve(int n);          // schedule + record buffers for n iterations
    void band_dev_forward_backward();  // iteration sched_pos: forward + backward on the band
    void band_dev_step();              // latent + NN Adam with the exchanged flags
    const Plan* device_plan() const { return d_plan_; }
    const LaunchCtx& launch_ctx() const { return L_; }
    int device() const { return device_; }

    // state transfer
    void set_state(const float* lat, const float* par, const float* lm, const float* lv,
                   const int64_t* lt, const float* nm, const float* nv, const int64_t* nt);
    void get_state(float* lat, float* par, float* lm, float* lv, int64_t* lt, float* nm,
                   float* nv, int64_t* nt);
    void get_grads(float* lg, float* pg);
    void soap_state(double* arena, float* m1, float* v2, int64_t* t, int64_t* n_arena);
    void set_soap_state(const double* arena, const float* m1, const float* v2, const int64_t* t);
    void set_q(const int32_t* q);
    void decode_terms(const float* params, int which, double* bits, double* mse);
    // (mu, sigma) of every quantised latent, params substituted (NULL: own)
    void latent_mu_sigma(const float* params, float* mu, float* sigma);
    void get_q(int32_t* q);
    void get_params(float* p);

    // geometry
    const Plan& plan() const { return H_; }
    const std::vector<TensorInfo>& tensors() const { return tensors_; }
    const std::vector<GridInfo>& grids() const { return grids_; }
    const cc_encoder_config& enc() const { return enc_; }
    const std::string& log_path() const { return log_path_; }
    bool loaded() const { return loaded_; }
    void synchronize();

private:
    void init(const float* image, int h, int w);
    void mark(int id, int on);  // 0 main, 1 side, 2 tail stream
    void nn_apply(const LaunchCtx& ctx, bool do_step, bool count_iter, bool log_rec);
    void build_plan();
    void allocate();
    void make_pad_maps();
    void require_loaded() const;
    void init_params_host(uint64_t stream, std::vector<float>& out) const;
    void enqueue_proxy(bool batched);
    void fork(bool tail = false);
    void join(bool tail = false);
    LaunchCtx side(bool tail = false) const;
    cudaStream_t branch(bool tail) const;  // side / tail stream (the main one under CCB_SERIAL=1)
    void enqueue_hardround(int slot);
    void enqueue_true_cost();
    void run_graph(int which, int slot = -1);
    cudaGraphExec_t ensure_graph(int which, int slot = -1);
    void read_scalars();
    void note_low_priority(cudaStream_t st);
    void apply_node_priorities(cudaGraph_t g);
    void ensure_snapshot(int slot);
    void zero_pads();
    void* dalloc(size_t bytes);

    cc_encoder_config enc_;
    cc_decoder_config dec_;
    std::string log_path_;
    int device_ = 0;
    int num_sms_ = 148;
    cudaStream_t stream_ = nullptr;
    cudaStream_t own_stream_ = nullptr;
    cudaStream_t side_stream_ = nullptr;  // concurrent rate branch
    cudaStream_t tail_stream_ = nullptr;  // concurrent fine-grid gradient tail
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    cudaEvent_t ev_fin_ = nullptr;    // k_finalize done (the cost flag the latent Adam step reads)
    cudaEvent_t ev_rate_ = nullptr;   // rate branch (ARM, dF pyramid) done
    cudaEvent_t ev_synfwd_ = nullptr; // synthesis forward + posts done (trunk weight grads may start)
    cudaEvent_t ev_sched_ = nullptr;  // the pinned schedule upload of the last batch
    Plan H_{};
    Plan* d_plan_ = nullptr;
    LaunchCtx L_{};
    bool armc_on_ = false;   // the constant-bank ARM's launch geometry (cc_armc.cuh)
    int armc_slot_ = -1;     // its constant slot (-1: none free, the FFMA2 tile kernel runs)


    std::vector<TensorInfo> tensors_;
    std::vector<GridInfo> grids_;
    std::vector<void*> allocs_;
    int4* d_tiles_ = nullptr;
    double* d_sched_ = nullptr;     // 3 doubles per iteration (batched)
    double* d_rec_ = nullptr;       // device mapping of h_rec_
    double* h_rec_ = nullptr;       // 4 doubles per iteration (batched), mapped pinned host memory
    double* h_sched_ = nullptr;     // pinned schedule staging
    float* d_param_save_ = nullptr; // decode_terms: the trainer's own parameters
    float* d_mu_sigma_ = nullptr;   // latent_mu_sigma output (mu | sigma)
    cudaEvent_t* tl_ev_ = nullptr;  // timeline marks while capturing ccb_timeline
    int sched_cap_ = 0;
    DevScalars* h_scal_ = nullptr;  // pinned mirror
    bool loaded_ = false;
    double cur_cost_ = 0.0;
    double last_mse_ = 0.0, last_bits_ = 0.0;
    std::map<int, CandSlot> cands_;
    std::map<int, SnapSlot> snaps_;
    // captured graphs: 0 proxy(single), 1 proxy(batched), 2 true_cost, 100+slot hardround
    std::map<int, cudaGraphExec_t> graphs_;
    struct Sizes {
        int64_t pad = 0, dctx = 0, dfeat = 0, ups = 0, partials = 0, z = 0, soap = 0;
    } sizes_;
    struct BandSpec {
        bool on = false;
        int hg = 0, r0 = 0, r1 = 0, halo = 0;
    } band_;
    std::vector<int4> tiles_host_;
    std::vector<int4> ifce_items_host_;  // k_ifce_dw work items (cc_arm.cu)
    std::vector<cudaGraphNode_t> low_nodes_;  // captured nodes to run at the least priority
};

// Several images of one geometry trained in lock-step by ONE set of launches
// per stage (BASELINE config 3: independent images batched within a GPU; the
// reference's only multi-image mode is independent encodes in a thread pool,
// tools/coolcodec.cpp:150-171).  Every trainer keeps its own buffers, state,
// counters and records; the batch owns the array of their device plans and the
// batched iteration graph, launched on the first trainer's stream (all
// trainers are moved onto it).
class Batch {
public:
    explicit Batch(std::vector<Trainer*> trainers);
    ~Batch();
    Batch(const Batch&) = delete;
    Batch& operator=(const Batch&) = delete;
    void reserve_iterations(int n);
    void enqueue_proxy_iterations(int n, const double* lr, const double* temp, const double* noise);
    void synchronize();
    int size() const { return int(t_.size()); }

private:
    std::vector<Trainer*> t_;
    Plan* d_plans_ = nullptr;
    std::vector<float*> stages_;  // each image's constant-bank ARM weight image (cc_armc.cuh)
    cudaGraphExec_t graph_ = nullptr;
    int cap_ = 0;
};

int64_t host_sync_count();  // host waits on the device issued by the library so far
void count_host_sync();

void fp32_peak(int device, double* tflops, double* ms);
void eval_math(int fn, int n, const float* a, const float* b, const float* c, float* out);
void gauss(uint64_t stream, uint64_t idx0, int n, float* out);

// warmup / train (encoder.hpp:315-413) over the B200 Trainer.
void warmup(Trainer& tr);
// train: with the host image (image != NULL) the warm-up candidates of each
// round run concurrently in helper trainers (warmup_batched).
void train(Trainer& tr, cc_train_stats* stats, const float* image = nullptr, int h = 0, int w = 0,
           const cc_decoder_config* dec = nullptr, int device = 0);
bool warmup_batched(Trainer& tr, const float* image, int h, int w, const cc_decoder_config& dec, int device);

}  // namespace ccb
