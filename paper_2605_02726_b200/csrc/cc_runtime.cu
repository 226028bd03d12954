// cc_runtime.cu — the B200 Trainer: geometry (build_latents latent.hpp:46-70,
// make_model model.hpp:80-123, make_context_offsets entropy_model.hpp:24-45),
// one device arena per image, and the per-iteration launch sequences captured
// once into CUDA graphs and replayed (no host work per kernel).
#include "cc_runtime.h"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>

#include "cc_math.cuh"

namespace ccb {

bool pdl_enabled(char which) {
    static const char* e = std::getenv("CCB_PDL");  // A/B: 0 off, f / b one direction only
    if (!e) return true;
    if (e[0] == '0') return false;
    if (e[0] == 'f' || e[0] == 'b') return which == e[0];
    return true;
}

void throw_config(const char* what) { throw ConfigError(what); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {

constexpr int kArmTileHost = kArmTile;
constexpr int kRMaxHost = 12;
constexpr int kFMaxHost = 8;
constexpr int kSnapSlots = 8;
constexpr float kBicubic[4] = {-0.0234375f, -0.0703125f, 0.2265625f, 0.8671875f};  // model.hpp:127

int ceil_div(int a, int b) { return (a + b - 1) / b; }

// make_context_offsets (entropy_model.hpp:24-45)
void context_offsets(int count, std::vector<int>& dy, std::vector<int>& dx, int& pad) {
    struct Cand {
        int d2, dy, dx;
    };
    std::vector<Cand> c;
    const int radius = 8;
    for (int y = -radius; y <= 0; ++y)
        for (int x = -radius; x <= radius; ++x) {
            if (y == 0 && x >= 0) continue;
            c.push_back({y * y + x * x, y, x});
        }
    std::sort(c.begin(), c.end(), [](const Cand& a, const Cand& b) {
        if (a.d2 != b.d2) return a.d2 < b.d2;
        if (a.dy != b.dy) return a.dy < b.dy;
        return a.dx < b.dx;
    });
    if (count > int(c.size())) throw ConfigError("spatial context too large");
    pad = 0;
    dy.clear();
    dx.clear();
    for (int i = 0; i < count; ++i) {
        dy.push_back(c[i].dy);
        dx.push_back(c[i].dx);
        pad = std::max({pad, -c[i].dy, std::abs(c[i].dx)});
    }
}

}  // namespace

Trainer::Trainer(const float* image, int h, int w, const cc_encoder_config& enc,
                 const cc_decoder_config& dec, int device)
    : enc_(enc), dec_(dec), device_(device) {
    init(image, h, w);
}

Trainer::Trainer(const float* image_window, int hg, int w, int r0, int r1, int halo,
                 const cc_encoder_config& enc, const cc_decoder_config& dec, int device)
    : enc_(enc), dec_(dec), device_(device) {
    int w0 = 0, w1 = 0;
    band_window(hg, w, r0, r1, halo, &w0, &w1);
    band_.on = true;
    band_.hg = hg;
    band_.r0 = r0;
    band_.r1 = r1;
    band_.halo = halo;
    init(image_window, w1 - w0, w);
}

void Trainer::init(const float* image, int h, int w) {
    const cc_encoder_config& enc = enc_;
    if (h < 1 || w < 1) throw ConfigError("image dimensions must be positive");
    log_path_ = enc.log_path ? enc.log_path : "";
    enc_.log_path = nullptr;

    H_.H = h;
    H_.W = w;
    CCB_CUDA(cudaSetDevice(device_));
    cudaDeviceProp prop;
    CCB_CUDA(cudaGetDeviceProperties(&prop, device_));
    if (prop.major < 10)
        throw CudaError("libcoolchic_b200 is built for sm_100a; device " + std::string(prop.name) +
                        " is sm_" + std::to_string(prop.major) + std::to_string(prop.minor));
    num_sms_ = prop.multiProcessorCount;
    {
        // main stream (the critical chain) at the greatest priority, the
        // concurrent branches at the least: effective for eager launches; a
        // CUDA graph runs its nodes at the launch stream's priority
        int lo = 0, hi = 0;
        CCB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CCB_CUDA(cudaStreamCreateWithPriority(&own_stream_, cudaStreamNonBlocking, hi));
        CCB_CUDA(cudaStreamCreateWithPriority(&side_stream_, cudaStreamNonBlocking, lo));
        CCB_CUDA(cudaStreamCreateWithPriority(&tail_stream_, cudaStreamNonBlocking, lo));
    }
    CCB_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    CCB_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    CCB_CUDA(cudaEventCreateWithFlags(&ev_sched_, cudaEventDisableTiming));
    CCB_CUDA(cudaEventCreateWithFlags(&ev_fin_, cudaEventDisableTiming));
    CCB_CUDA(cudaEventCreateWithFlags(&ev_rate_, cudaEventDisableTiming));
    CCB_CUDA(cudaEventCreateWithFlags(&ev_synfwd_, cudaEventDisableTiming));
    stream_ = own_stream_;
    build_plan();
    allocate();
    upload_image(image);
}

Trainer::~Trainer() {
    cudaSetDevice(device_);
    // a trainer moved onto another's stream (a batch) must not touch that
    // stream here: its owner may be gone already
    if (stream_ && stream_ == own_stream_) cudaStreamSynchronize(stream_);
    else if (stream_) cudaDeviceSynchronize();
    armc_release_slot(armc_slot_);
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
    for (auto& kv : cands_) {
        for (float* p : {kv.second.y, kv.second.m, kv.second.v, kv.second.p, kv.second.nm, kv.second.nv})
            cudaFree(p);
        if (kv.second.soap) cudaFree(kv.second.soap);
    }
    for (auto& kv : snaps_) {
        cudaFree(kv.second.y);
        cudaFree(kv.second.p);
    }
    for (void* p : allocs_) cudaFree(p);
    if (h_scal_) cudaFreeHost(h_scal_);
    if (d_sched_) cudaFree(d_sched_);
    if (h_rec_) cudaFreeHost(h_rec_);  // d_rec_ is its device mapping
    if (h_sched_) cudaFreeHost(h_sched_);
    if (side_stream_) cudaStreamSynchronize(side_stream_);
    if (tail_stream_) cudaStreamSynchronize(tail_stream_);
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (ev_sched_) cudaEventDestroy(ev_sched_);
    if (ev_fin_) cudaEventDestroy(ev_fin_);
    if (ev_rate_) cudaEventDestroy(ev_rate_);
    if (ev_synfwd_) cudaEventDestroy(ev_synfwd_);
    if (side_stream_) cudaStreamDestroy(side_stream_);
    if (tail_stream_) cudaStreamDestroy(tail_stream_);
    if (own_stream_) cudaStreamDestroy(own_stream_);
}

void* Trainer::dalloc(size_t bytes) {
    void* p = nullptr;
    CCB_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    CCB_CUDA(cudaMemset(p, 0, std::max<size_t>(bytes, 16)));
    allocs_.push_back(p);
    return p;
}

// Row bands: own full-resolution rows [r0, r1) of an image
// of hg rows; every grid holds its own rows plus `halo` rows on each side
// (clipped at the image border).  band_window gives the pixel rows to upload.
void Trainer::band_window(int hg, int w, int r0, int r1, int halo, int* w0, int* w1) {
    const int L = int64_t(hg) * int64_t(w) < 1000000 ? 7 : 8;
    const int align = 1 << (L - 1);
    if (hg < 1 || w < 1 || r0 < 0 || r1 > hg || r0 >= r1)
        throw ConfigError("band rows must satisfy 0 <= r0 < r1 <= H");
    if (r0 % align != 0 || (r1 != hg && r1 % align != 0))
        throw ConfigError("band edges must be multiples of 2^(L-1) (or the image height)");
    // 6 rows per level keep every own row exact: the ARM context reaches 3 rows
    // up, an upsampling cascade loses < 6 rows per level to the window edge
    // and the synthesis posts reach 4 pixel rows
    if (halo < 6) throw ConfigError("band halo must be >= 6 rows");
    *w0 = std::max(0, r0 - halo);
    *w1 = std::min(hg, r1 + halo);
}

void Trainer::build_plan() {
    Plan& P = H_;
    const int h = P.H, w = P.W;
    const int hg = band_.on ? band_.hg : h;           // global image rows
    P.L = int64_t(hg) * int64_t(w) < 1000000 ? 7 : 8;  // latent_levels, config.hpp:84
    P.hyper = dec_.use_hyperlatents ? P.L - 4 : 0;     // kHyperCoarsestLevel = 4
    P.S = dec_.spatial_ctx;
    P.F = dec_.ifce_dim;
    P.D = P.S + P.F;
    P.Wd = dec_.arm_width;
    P.syn_F = dec_.synth_hidden;
    P.posts = dec_.synth_posts;
    P.use_stab_arm = dec_.use_stabilizer;
    P.use_stab_syn = dec_.use_stabilizer;
    if (P.S < 0 || P.F < 0 || P.Wd < 1 || P.syn_F < 1)
        throw ConfigError("decoder dimensions must be positive");
    if (P.S > kMaxCtx) throw ConfigError("spatial context too large for the B200 kernels");
    if (P.F > kFMaxHost) throw ConfigError("ifce_dim > 8 is not supported by the B200 kernels");
    if (P.D < 1) throw ConfigError("ARM input dimension must be positive");
    arm_padded_dims(P.D, P.Wd, &P.Dp, &P.Wp);
    if (P.Dp < 0) throw ConfigError("ARM dims (input <= 40, width <= 40) exceeded");
    if (band_.on && !arm_uses_v2(P.Dp, P.Wp))
        throw ConfigError("row bands need the register-tiled ARM kernel (ARM input/width <= 32/28)");
    if (syn_padded_hidden(P.syn_F) < 0) throw ConfigError("synth_hidden > 64 is not supported");
    if (P.posts < 0 || P.posts > 2) throw ConfigError("synth_posts must be 0, 1 or 2");
    P.npix = int64_t(h) * w;
    P.npix_global = int64_t(hg) * w;
    P.band = band_.on ? 1 : 0;
    P.lambda = enc_.lambda;
    P.seed = enc_.seed;
    P.rate_upstream = float(enc_.lambda / double(P.npix_global));  // encoder.hpp:64

    std::vector<int> dy, dx;
    int cpad = 0;
    context_offsets(P.S, dy, dx, cpad);
    for (int o = 0; o < P.S; ++o) {
        P.ctx_dy[o] = dy[o];
        P.ctx_dx[o] = dx[o];
    }
    P.P = std::max(1, cpad);  // encoder.hpp:218
    // the register-tiled ARM stages a (P+1)-row context window of <= 4-wide
    // halo; every context that fits its input width (<= 32) has P <= 4
    if (arm_uses_v2(P.Dp, P.Wp) && P.P > 4)
        throw ConfigError("spatial context halo > 4 exceeds the register-tiled ARM window");

    // ---- grids in decode order (latent.hpp:66-68) ----
    struct G {
        int level, hyper;
    };
    std::vector<G> order;
    for (int k = P.L - 1; k >= 4 && dec_.use_hyperlatents; --k) order.push_back({k, 1});
    for (int k = P.L - 1; k >= 0; --k) order.push_back({k, 0});
    P.n_grids = int(order.size());
    if (P.n_grids > kMaxGrids) throw ConfigError("too many grids");
    int64_t pad_cur = 0, lat_cur = 0, dctx_cur = 0;
    // context-gradient row partials (cc_ctx.cuh) instead of S planes: 3.3x less
    // dctx traffic and a cheaper gather (tail 69 -> 63 us), but the partial
    // sums cost the ARM more than that (263 -> 283-291 us alone, 0.453 ->
    // 0.465-0.472 ms per iteration at 512x768): opt-in, CCB_CTX_PART=1
    static const bool ctx_part_env = [] {
        const char* e = std::getenv("CCB_CTX_PART");
        return e && e[0] == '1';
    }();
    P.ctx_part = (ctx_part_env && arm_uses_v2(P.Dp, P.Wp)) ? 1 : 0;
    // the constant-bank ARM (cc_armc.cuh) where it instantiates the dims; its
    // launch geometry (kArmcPerSm x 64-thread CTAs per SM) sizes the ARM's
    // partial rows even when no constant slot is free (then the FFMA2 tile
    // kernel runs on the same grid)
    armc_on_ = armc_supported(P.Dp, P.Wp) && !P.ctx_part;
    for (int i = 0; i < kMaxLevels; ++i) P.main_gi[i] = -1;
    for (int gi = 0; gi < P.n_grids; ++gi) {
        GridGeom& g = P.g[gi];
        g.level = order[gi].level;
        g.hyper = order[gi].hyper;
        g.grows = ceil_div(hg, 1 << g.level);
        g.cols = ceil_div(w, 1 << g.level);
        {
            int o0 = 0, o1 = g.grows, w0 = 0, w1 = g.grows;
            if (band_.on) {
                o0 = band_.r0 >> g.level;
                o1 = band_.r1 == hg ? g.grows : band_.r1 >> g.level;
                w0 = std::max(0, o0 - band_.halo);
                w1 = std::min(g.grows, o1 + band_.halo);
            }
            g.row0 = w0;
            g.rows = w1 - w0;
            g.own_lo = o0 - w0;
            g.own_hi = o1 - w0;
        }
        // row stride rounded to 16 bytes: every grid's padded array is a
        // valid TMA tensor (16-byte aligned base and row pitch; the extra
        // columns belong to the zero border)
        g.stride = (g.cols + 2 * P.P + 3) & ~3;
        g.pad_base = pad_cur + int64_t(P.P) * g.stride + P.P;
        pad_cur += int64_t(g.rows + 2 * P.P) * g.stride;
        g.lat_off = lat_cur;
        lat_cur += int64_t(g.rows) * g.cols;
        g.dctx_off = dctx_cur;
        if (P.ctx_part)  // [row][d = 0..P][row tile][kArmTile + 2P]
            dctx_cur += int64_t(g.rows) * (P.P + 1) * ceil_div(g.cols, kArmTileHost) * (kArmTileHost + 2 * P.P);
        else
            dctx_cur += int64_t(P.S) * g.rows * g.cols;
        g.main_level = g.hyper ? -1 : g.level;
        if (!g.hyper) P.main_gi[g.level] = gi;
        g.ifce_slot = -1;
        g.rdim = 0;
        g.dfeat_off = 0;
        grids_.push_back({g.level, g.hyper, g.rows, g.cols, g.lat_off, -1});
    }
    P.n_latents = lat_cur;
    {
        const GridGeom& g0 = P.g[P.main_gi[0]];
        if (g0.rows != h) throw ConfigError("internal: band pixel window does not match grid 0");
        P.pix_row0 = g0.row0;
        P.pix_own_lo = g0.own_lo;
        P.pix_own_hi = g0.own_hi;
    }

    // ---- IFCE slots (model.hpp:94-101): main levels 0..min(3,L)-1 ----
    P.n_slots = 0;
    int64_t df_cur = 0;
    if (P.F > 0) {
        for (int k = 0; k < std::min(3, P.L); ++k) {
            const int s = P.n_slots++;
            const int gi = P.main_gi[k];
            GridGeom& g = P.g[gi];
            g.ifce_slot = s;
            g.rdim = P.hyper + (P.L - 1 - k);  // ifce_source_count, model.hpp:70-71
            if (g.rdim > 11) throw ConfigError("IFCE source count above 11 (at most 8 latent levels)");
            if (g.rdim > kRMaxHost) throw ConfigError("IFCE source count exceeds 12");
            if (g.rdim != gi) throw ConfigError("internal: IFCE sources must precede the grid");
            grids_[gi].ifce_slot = s;
            P.slot_gi[s] = gi;
            P.slot_smax[s] = (P.L - 1) - k;
            // pyramid blocks are aligned to global rows: origin A (multiple of 2^smax)
            const int A = (g.row0 >> P.slot_smax[s]) << P.slot_smax[s];
            P.slot_pyr_a[s] = A;
            int cc = g.cols;
            for (int l = 0; l <= P.slot_smax[s]; ++l) {
                if (l > 0) cc = ceil_div(cc, 2);
                const int rr = l == 0 ? g.rows : ceil_div(g.row0 + g.rows - A, 1 << l);
                P.slot_pyr_rows[s][l] = rr;
                P.slot_pyr_cols[s][l] = cc;
                P.slot_pyr_off[s][l] = df_cur;
                df_cur += int64_t(P.F) * rr * cc;
            }
            g.dfeat_off = P.slot_pyr_off[s][0];
        }
    }

    // ---- parameters in for_each_param order (model.hpp:158-171) ----
    int off = 0;
    auto add = [&](const std::string& name, int rows, int cols) {
        TensorInfo t{name, rows, cols, rows * cols, off};
        tensors_.push_back(t);
        off += rows * cols;
        return t.offset;
    };
    const int D = P.D, Wd = P.Wd;
    P.off_l1w = add("arm.l1.w", Wd, D);
    P.off_l1b = add("arm.l1.b", 1, Wd);
    P.off_l2w = add("arm.l2.w", Wd, Wd);
    P.off_l2b = add("arm.l2.b", 1, Wd);
    P.off_hw = add("arm.head.w", 2, Wd);
    P.off_hb = add("arm.head.b", 1, 2);
    P.off_astab = dec_.use_stabilizer ? add("arm.stab", 2, D) : -1;
    for (int s = 0; s < P.n_slots; ++s) {
        const int rd = P.g[P.slot_gi[s]].rdim;
        P.off_ifw[s] = add("ifce" + std::to_string(s) + ".w", P.F, rd);
        P.off_ifb[s] = add("ifce" + std::to_string(s) + ".b", 1, P.F);
    }
    for (int j = 0; j < P.L - 1; ++j) {
        P.off_tconv[j] = add("ups" + std::to_string(j) + ".tconv", 1, 4);
        P.off_refine[j] = add("ups" + std::to_string(j) + ".refine", 1, 3);
    }
    P.off_c1w = add("syn.c1.w", P.syn_F, P.L);
    P.off_c1b = add("syn.c1.b", 1, P.syn_F);
    P.off_c2w = add("syn.c2.w", 3, P.syn_F);
    P.off_c2b = add("syn.c2.b", 1, 3);
    for (int i = 0; i < P.posts; ++i) P.off_pw[i] = add("syn.post" + std::to_string(i) + ".w", 3, 27);
    for (int i = 0; i < P.posts; ++i) P.off_pb[i] = add("syn.post" + std::to_string(i) + ".b", 1, 3);
    P.off_sstab = dec_.use_stabilizer ? add("syn.stab", 3, P.L) : -1;
    P.n_params = off;
    P.n_tensors = int(tensors_.size());
    if (P.n_tensors > kMaxTensors) throw ConfigError("too many tensors");
    P.use_soap = enc_.use_soap ? 1 : 0;
    P.soap_dmax = 1;
    P.soap_nmax = 1;
    int64_t soap_cur = 0;
    for (int t = 0; t < P.n_tensors; ++t) {
        P.tensor_off[t] = tensors_[t].offset;
        P.tensor_size[t] = tensors_[t].size;
        P.tensor_rows[t] = tensors_[t].rows;
        P.tensor_cols[t] = tensors_[t].cols;
        P.soap_off[t] = soap_cur;
        const int r = tensors_[t].rows, c = tensors_[t].cols;
        soap_cur += 2 * int64_t(r) * r + 2 * int64_t(c) * c;
        P.soap_dmax = std::max(P.soap_dmax, std::max(r, c));
        P.soap_nmax = std::max(P.soap_nmax, r * c);
    }
    sizes_.soap = P.use_soap ? soap_cur : 0;
    if (P.use_soap && soap_smem(P) > 227 * 1024)
        throw ConfigError("SOAP: a parameter matrix is too large for the on-chip step");

    // ---- upsampling stages (synthesis.hpp:66-92) ----
    // Cascade k runs on rows aligned to its latent window: level j holds
    // global rows [row0_k << (k-j), end_j) (the image end at the bottom band),
    // so every stage is a plain 2x upsampling of a sub-image; its level-0
    // output (z plane k) is taller than the pixel window, which it contains.
    int64_t ub = 0;
    int64_t stage_out_off[kMaxLevels][kMaxLevels];  // [k][j]
    int64_t zcur = int64_t(h) * w;                  // z plane 0 = grid 0 copy
    P.zpix[0] = 0;
    for (int j = 0; j < kMaxLevels; ++j) P.ups_n[j] = 0;
    for (int k = 1; k < P.L; ++k) {
        const GridGeom& gk = P.g[P.main_gi[k]];
        const bool bottom = gk.row0 + gk.rows == gk.grows;
        auto lvl_start = [&](int j) { return gk.row0 << (k - j); };
        auto lvl_end = [&](int j) { return bottom ? ceil_div(hg, 1 << j) : (gk.row0 + gk.rows) << (k - j); };
        for (int j = k - 1; j >= 0; --j) {
            UpsStage& st = P.ups[j][P.ups_n[j]++];
            st.k = k;
            st.rows_in = lvl_end(j + 1) - lvl_start(j + 1);
            st.cols_in = ceil_div(w, 1 << (j + 1));
            st.rows_out = lvl_end(j) - lvl_start(j);
            st.cols_out = ceil_div(w, 1 << j);
            if (st.rows_out > 2 * st.rows_in || st.rows_out < 1)
                throw ConfigError("internal: inconsistent upsampling window");
            if (j == k - 1) {
                const GridGeom& g = P.g[P.main_gi[k]];
                st.in_is_pad = 1;
                st.in_off = g.pad_base;
                st.in_stride = g.stride;
            } else {
                st.in_is_pad = 0;
                st.in_off = stage_out_off[k][j + 1];
                st.in_stride = st.cols_in;
            }
            st.row_off = ub;
            ub += int64_t(st.rows_in) * st.cols_out;
            st.col_off = ub;
            ub += int64_t(st.rows_out) * st.cols_out;
            if (j == 0) {
                st.out_is_z = 1;
                st.out_off = zcur;
                const int zoff = P.pix_row0 - lvl_start(0);
                if (zoff < 0 || zoff + h > st.rows_out)
                    throw ConfigError("internal: z plane does not cover the pixel window");
                P.zpix[k] = zcur + int64_t(zoff) * w;
                zcur += int64_t(st.rows_out) * st.cols_out;
            } else {
                st.out_is_z = 0;
                st.out_off = ub;
                ub += int64_t(st.rows_out) * st.cols_out;
            }
            stage_out_off[k][j] = st.out_off;
            // backward wiring
            st.dout_is_z = j == 0;
            st.dout_off = st.out_off;  // dz plane k, or ups_grad at the same offset
            st.din_is_lat = j == k - 1;
            st.din_off = st.din_is_lat ? P.g[P.main_gi[k]].lat_off : stage_out_off[k][j + 1];
        }
    }
    // stage (k, j+1)'s output offset is known before stage (k, j) is built
    // because stages are created from j = k-1 downward.
    const int64_t ups_total = ub;
    sizes_.z = zcur;
    P.zvec = (P.npix % 4 == 0) ? 1 : 0;
    for (int k = 0; k < P.L; ++k)
        if (P.zpix[k] % 4 != 0) P.zvec = 0;

    // ---- launch geometry ----
    L_.num_sms = num_sms_;
    auto cap = [&](int64_t n, int per) {
        int64_t b = (n + per - 1) / per;
        b = std::min<int64_t>(b, int64_t(num_sms_) * 8);
        return int(std::max<int64_t>(b, 1));
    };
    L_.elem_blocks = cap(P.n_latents, 256);
    L_.pix_blocks = cap(P.npix, 256);
    L_.red_blocks = num_sms_;
    // ARM tiles: row segments of <= 128 latents (grid, first latent, row,
    // length), so a tile's causal context is one (P+1)-row window and its
    // IFCE sources are one segment per coarser grid
    std::vector<int4> tiles;
    for (int gi = 0; gi < P.n_grids; ++gi)
        for (int r = 0; r < P.g[gi].rows; ++r)
            for (int c0 = 0; c0 < P.g[gi].cols; c0 += kArmTileHost)
                tiles.push_back(make_int4(gi, r * P.g[gi].cols + c0, r, std::min(kArmTileHost, P.g[gi].cols - c0)));
    L_.arm_ntiles = int(tiles.size());
    int arm_occ = arm_blocks_per_sm(P.Dp, P.Wp);
    if (const char* e = std::getenv("CCB_ARM_OCC")) arm_occ = std::max(1, std::min(arm_occ, std::atoi(e)));
    // 1.5 CTAs per SM when 2 fit: the persistent ARM then leaves CTA slots on
    // half the SMs to the concurrent distortion branch (measured: 0.558 ->
    // 0.542 ms per iteration at 512x768 vs 2 per SM)
    // (the tensor-core kernel runs 2 x 128-thread CTAs per SM: the second
    // CTA's work overlaps the first one's tensor-core round trips)
    L_.arm_blocks = std::min(L_.arm_ntiles, arm_uses_tc(P.Dp, P.Wp)  ? num_sms_ * arm_occ
                                            : arm_occ >= 2          ? num_sms_ * 3 / 2
                                                                    : num_sms_ * arm_occ);
    if (armc_on_) {
        // 3.25 CTAs per SM when 4 fit: the free slots on three quarters of
        // the SMs let the concurrent distortion branch (the critical chain)
        // run its kernels beside the ARM (512x768, the kernel at <= 168
        // registers: 4 per SM 0.439 ms per iteration, 3.5 0.420, 3.25 0.413,
        // 3 0.424)
        int per4 = 4 * armc_blocks_per_sm(P.Dp, P.Wp);
        if (per4 >= 16) per4 = 13;
        if (const char* e = std::getenv("CCB_ARMC_OCC")) per4 = 4 * std::max(1, std::min(per4 / 4, std::atoi(e)));
        L_.arm_blocks = std::min(L_.arm_ntiles, num_sms_ * per4 / 4);
    }
    if (const char* e = std::getenv("CCB_ARM_CTAS"))  // A/B: explicit persistent CTA count
        L_.arm_blocks = std::max(1, std::min(L_.arm_ntiles, std::atoi(e)));
    const int FP = syn_padded_hidden(P.syn_F);
    const int64_t syn_tiles = (P.npix + kSynTile - 1) / kSynTile;
    const int syn_per_sm = syn_trunk_blocks_per_sm(FP);
    L_.syn_ntiles = int(syn_tiles);
    L_.syn_blocks = int(std::min<int64_t>(syn_tiles, int64_t(num_sms_) * syn_per_sm));
    P.n_bits_part = L_.arm_blocks;
    // k_syn_post: persistent, one 16x16 tile at a time, one MSE/post-grad row per CTA
    P.n_mse_part = std::max(1, std::min(syn_post_tiles(h, w), 3 * num_sms_));

    // ---- partial regions ----
    int64_t pbase = 0;
    P.n_regions = 0;
    auto region = [&](int param_off, int count, int nblocks) {
        const int r = P.n_regions++;
        if (r >= kMaxPartialRegions) throw ConfigError("too many partial regions");
        P.region[r] = PartialRegion{param_off, count, nblocks, pbase};
        pbase += int64_t(count) * nblocks;
        return r;
    };
    // constant-bank ARM: the IFCE weight gradients come from k_ifce_dw (its
    // own partial rows); the ARM's region then ends before them
    P.ifce_sep = (armc_on_ && P.n_slots > 0 && P.F > 0) ? 1 : 0;
    P.arm_nvals = P.ifce_sep ? P.off_ifw[0] : P.off_tconv[0];
    P.reg_arm = region(0, P.arm_nvals, L_.arm_blocks);
    for (int s = 0; s < kMaxSlots; ++s) P.reg_ifce[s] = -1;
    P.n_ifce_items = 0;
    ifce_items_host_.clear();
    if (P.ifce_sep) {
        ifce_items_host_ = ifce_dw_items(P, P.ifce_item0);
        P.n_ifce_items = int(ifce_items_host_.size());
        for (int s = 0; s < P.n_slots; ++s) {
            const int rd = P.g[P.slot_gi[s]].rdim;
            if (P.off_ifb[s] != P.off_ifw[s] + P.F * rd) throw ConfigError("IFCE parameters are not contiguous");
            const int end = s + 1 < P.n_slots ? P.ifce_item0[s + 1] : P.n_ifce_items;
            P.reg_ifce[s] = region(P.off_ifw[s], P.F * rd + P.F, end - P.ifce_item0[s]);
        }
    }
    P.ups_jc = ups_coarse_from(P);
    for (int j = 0; j < P.L - 1; ++j) {
        // k_ups_bwd writes one row per CTA: dk4 (row + column passes) and dr3;
        // fused coarse stages one row per cascade
        const int nb = j >= P.ups_jc ? ups_chain_ctas() * P.ups_n[j]
                                     : ups_blocks_x(P, j, num_sms_, false) * P.ups_n[j];
        P.reg_ups_rows[j] = region(P.off_tconv[j], 4, nb);
        P.reg_ups_cols[j] = -1;
        P.reg_ups_ref[j] = region(P.off_refine[j], 3, nb);
    }
    P.syn_nvals = P.n_params - P.off_c1w;
    P.reg_syn_trunk = region(P.off_c1w, P.syn_nvals, L_.syn_blocks);
    for (int i = 0; i < P.posts; ++i)
        P.reg_post[i] = region(P.off_pw[0], P.off_pb[P.posts - 1] + 3 - P.off_pw[0], P.n_mse_part);

    // sizes for allocate()
    P.g[0].dfeat_off = P.g[0].dfeat_off;  // (no-op; keeps field initialised)
    allocs_.reserve(64);
    // stash sizes in the (otherwise unused before allocation) pointer fields via locals
    sizes_.pad = pad_cur;
    sizes_.dctx = dctx_cur;
    sizes_.dfeat = std::max<int64_t>(df_cur, 1);
    sizes_.ups = std::max<int64_t>(ups_total, 1);
    sizes_.partials = std::max<int64_t>(pbase, 1);
    tiles_host_ = tiles;
}

// One TMA descriptor per grid over its zero-bordered padded array
// ((rows + 2P) x stride fp32): the ARM loads a tile's causal-context window
// (P + 1 rows x kArmWinCols columns, zero fill past the array) with one
// cp.async.bulk.tensor instead of per-thread 4-byte copies.
void Trainer::make_pad_maps() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CCB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    Plan& P = H_;
    std::vector<CUtensorMap> maps(kMaxGrids);
    std::memset(maps.data(), 0, sizeof(CUtensorMap) * maps.size());
    for (int gi = 0; gi < P.n_grids; ++gi) {
        const GridGeom& g = P.g[gi];
        float* base = P.yhat_pad + g.pad_base - int64_t(P.P) * g.stride - P.P;
        const cuuint64_t dims[2] = {cuuint64_t(g.stride), cuuint64_t(g.rows + 2 * P.P)};
        const cuuint64_t strides[1] = {cuuint64_t(g.stride) * sizeof(float)};
        const cuuint32_t box[2] = {cuuint32_t(kArmWinCols), cuuint32_t(P.P + 1)};
        const cuuint32_t estr[2] = {1, 1};
        const CUresult r = encode(&maps[size_t(gi)], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed for grid " + std::to_string(gi));
    }
    auto* d = static_cast<CUtensorMap*>(dalloc(sizeof(CUtensorMap) * maps.size()));
    CCB_CUDA(cudaMemcpy(d, maps.data(), sizeof(CUtensorMap) * maps.size(), cudaMemcpyHostToDevice));
    P.pad_maps = d;
}

void Trainer::allocate() {
    Plan& P = H_;
    const int64_t nl = P.n_latents, np = P.npix;
    auto f32 = [&](int64_t n) { return static_cast<float*>(dalloc(sizeof(float) * size_t(n))); };
    P.yhat_pad = f32(sizes_.pad);
    make_pad_maps();
    P.y = f32(nl);
    P.lat_m = f32(nl);
    P.lat_v = f32(nl);
    P.lat_g = f32(nl);
    P.th1 = f32(nl);
    P.th2 = f32(nl);
    P.gown = f32(nl);
    P.dups = f32(nl);
    P.q = static_cast<int32_t*>(dalloc(sizeof(int32_t) * size_t(nl)));
    P.dctx = f32(std::max<int64_t>(sizes_.dctx, 1));
    P.dfeat = f32(sizes_.dfeat);
    P.z = f32(sizes_.z);
    P.dz = f32(sizes_.z);  // rows outside the pixel window stay zero
    P.ups_buf = f32(sizes_.ups);
    P.ups_grad = f32(sizes_.ups);
    P.ups_grad2 = nullptr;
    P.image = f32(3 * np);
    P.syn_t = f32(3 * np);
    P.syn_p[0] = f32(3 * np);
    P.syn_p[1] = f32(3 * np);
    P.syn_sz = f32(3 * np);
    P.syn_dx = f32(3 * np);
    P.syn_dt = f32(3 * np);
    P.syn_dtmp = f32(3 * np);
    P.params = f32(P.n_params);
    P.grads = f32(P.n_params);
    P.grads_d = static_cast<double*>(dalloc(sizeof(double) * size_t(P.n_params)));
    P.soap = P.use_soap ? static_cast<double*>(dalloc(sizeof(double) * size_t(sizes_.soap))) : nullptr;
    P.noise_buf = f32(nl);
    // k_syn_post2's fp64 flush slots, only when a CTA walks >= 16 tiles
    P.post_scratch = syn_post_tiles(P.H, P.W) >= 16 * P.n_mse_part
                         ? static_cast<double*>(dalloc(sizeof(double) * size_t(P.n_mse_part) * 256 * 30))
                         : nullptr;
    P.nn_m = f32(P.n_params);
    P.nn_v = f32(P.n_params);
    P.partials = static_cast<double*>(dalloc(sizeof(double) * size_t(sizes_.partials)));
    P.bc_lat = static_cast<double*>(dalloc(sizeof(double) * 2 * kMaxGrids));
    P.bits_part = static_cast<double*>(dalloc(sizeof(double) * size_t(P.n_bits_part)));
    P.mse_part = static_cast<double*>(dalloc(sizeof(double) * size_t(P.n_mse_part)));
    P.lat_t = static_cast<int64_t*>(dalloc(sizeof(int64_t) * kMaxGrids));
    P.nn_t = static_cast<int64_t*>(dalloc(sizeof(int64_t) * kMaxTensors));
    P.lat_ok = static_cast<int*>(dalloc(sizeof(int) * kMaxGrids));
    P.tensor_ok = static_cast<int*>(dalloc(sizeof(int) * kMaxTensors));
    P.scal = static_cast<DevScalars*>(dalloc(sizeof(DevScalars)));
    d_tiles_ = static_cast<int4*>(dalloc(sizeof(int4) * tiles_host_.size()));
    CCB_CUDA(cudaMemcpy(d_tiles_, tiles_host_.data(), sizeof(int4) * tiles_host_.size(),
                        cudaMemcpyHostToDevice));
    P.arm_cstage = armc_on_ ? f32(kArmcSlotFloats) : nullptr;
    P.ifce_items = nullptr;
    if (!ifce_items_host_.empty()) {
        int4* d = static_cast<int4*>(dalloc(sizeof(int4) * ifce_items_host_.size()));
        CCB_CUDA(cudaMemcpy(d, ifce_items_host_.data(), sizeof(int4) * ifce_items_host_.size(),
                            cudaMemcpyHostToDevice));
        P.ifce_items = d;
    }
    if (armc_on_) armc_slot_ = armc_acquire_slot();
    d_plan_ = static_cast<Plan*>(dalloc(sizeof(Plan)));
    CCB_CUDA(cudaMemcpy(d_plan_, &H_, sizeof(Plan), cudaMemcpyHostToDevice));
    CCB_CUDA(cudaMallocHost(&h_scal_, sizeof(DevScalars)));
    std::memset(h_scal_, 0, sizeof(DevScalars));
    for (int s = 0; s < kSnapSlots; ++s) h_scal_->snap_cost[s] = std::numeric_limits<double>::infinity();
    h_scal_->noise_iter = -1;  // nothing drawn ahead yet
    CCB_CUDA(cudaMemcpy(P.scal, h_scal_, sizeof(DevScalars), cudaMemcpyHostToDevice));

    L_.plan = d_plan_;
    L_.host = &H_;
    L_.stream = stream_;
    L_.arm_tiles = d_tiles_;
    L_.arm_cslot = armc_slot_;
    L_.arm_cstages = &H_.arm_cstage;
    arm_configure(P.Dp, P.Wp);
    if (armc_on_) armc_configure(P.Dp, P.Wp);
    syn_configure(syn_padded_hidden(P.syn_F));
    ups_configure();
    syn_post_configure();
    pyramid_configure(H_);
    if (P.use_soap) soap_configure(H_);
}

// host waits on the device issued by the library (ccb_host_sync_count)
static std::atomic<int64_t> g_host_syncs{0};
int64_t host_sync_count() { return g_host_syncs.load(); }
void count_host_sync() { g_host_syncs.fetch_add(1); }

void Trainer::synchronize() {
    count_host_sync();
    CCB_CUDA(cudaStreamSynchronize(stream_));
}

void Trainer::upload_image(const float* image) {
    CCB_CUDA(cudaSetDevice(device_));
    CCB_CUDA(cudaMemcpyAsync(H_.image, image, sizeof(float) * 3 * size_t(H_.npix),
                             cudaMemcpyHostToDevice, stream_));
    synchronize();
}

void Trainer::require_loaded() const {
    if (!loaded_) throw StateError("no candidate loaded (call fresh_candidate/load_candidate)");
}

void Trainer::zero_pads() {
    CCB_CUDA(cudaMemsetAsync(H_.yhat_pad, 0, sizeof(float) * size_t(sizes_.pad), stream_));
}

// init_model (model.hpp:137-156) — host side, bit-exact with the reference's
// contracted counter_uniform.
void Trainer::init_params_host(uint64_t stream, std::vector<float>& out) const {
    const Plan& P = H_;
    out.assign(size_t(P.n_params), 0.0f);
    uint64_t ctr = 0;
    auto sub = [&]() { return hash_combine(stream, ctr++); };
    auto kaiming = [&](int off, int n, int fan_in, uint64_t s) {
        const float a = std::sqrt(6.0f / float(fan_in));
        for (int i = 0; i < n; ++i) out[size_t(off + i)] = counter_uniform(s, uint64_t(i), -a, a);
    };
    kaiming(P.off_l1w, P.Wd * P.D, P.D, sub());
    kaiming(P.off_l2w, P.Wd * P.Wd, P.Wd, sub());
    kaiming(P.off_hw, 2 * P.Wd, P.Wd, sub());
    for (int s = 0; s < P.n_slots; ++s) {
        const int rd = P.g[P.slot_gi[s]].rdim;
        kaiming(P.off_ifw[s], P.F * rd, rd, sub());
    }
    for (int j = 0; j < P.L - 1; ++j) {
        for (int i = 0; i < 4; ++i) out[size_t(P.off_tconv[j] + i)] = kBicubic[i];
        out[size_t(P.off_refine[j])] = 1.0f;
    }
    kaiming(P.off_c1w, P.syn_F * P.L, P.L, sub());
    kaiming(P.off_c2w, 3 * P.syn_F, P.syn_F, sub());
}

void Trainer::fresh_candidate(int index) {
    CCB_CUDA(cudaSetDevice(device_));
    launch_init_latents(L_, hash_combine(enc_.seed, uint64_t(0x1000 + index)), 0.3f);
    std::vector<float> prm;
    init_params_host(hash_combine(enc_.seed, uint64_t(0x2000 + index)), prm);
    CCB_CUDA(cudaMemcpyAsync(H_.params, prm.data(), sizeof(float) * prm.size(),
                             cudaMemcpyHostToDevice, stream_));
    loaded_ = true;
    reset_optimizers();
    zero_pads();
    cur_cost_ = std::numeric_limits<double>::infinity();
    synchronize();
}

void Trainer::reset_optimizers() {
    require_loaded();
    const size_t nl = size_t(H_.n_latents), np = size_t(H_.n_params);
    CCB_CUDA(cudaMemsetAsync(H_.lat_m, 0, sizeof(float) * nl, stream_));
    CCB_CUDA(cudaMemsetAsync(H_.lat_v, 0, sizeof(float) * nl, stream_));
    CCB_CUDA(cudaMemsetAsync(H_.nn_m, 0, sizeof(float) * np, stream_));
    CCB_CUDA(cudaMemsetAsync(H_.nn_v, 0, sizeof(float) * np, stream_));
    CCB_CUDA(cudaMemsetAsync(H_.lat_t, 0, sizeof(int64_t) * kMaxGrids, stream_));
    CCB_CUDA(cudaMemsetAsync(H_.nn_t, 0, sizeof(int64_t) * kMaxTensors, stream_));
    if (H_.use_soap) launch_soap_reset(L_);  // SoapState::init (optim.hpp:130-143)
}

// NN-parameter optimizer step: Adam, or SOAP when EncoderConfig::use_soap
// (NnOptimizer::step, optim.hpp:277-286).
void Trainer::nn_apply(const LaunchCtx& ctx, bool do_step, bool count_iter, bool log_rec) {
    if (H_.use_soap)
        launch_soap_apply(ctx, do_step, count_iter, log_rec);
    else
        launch_nn_apply(ctx, do_step, count_iter, log_rec);
}

// ---------------------------------------------------------------- sequences
// Trainer::proxy_iteration (encoder.hpp:97-135)
// The rate branch (ARM + IFCE, dF pyramid) and the distortion branch
// (upsampling, synthesis, their backward) only share ŷ as input, so they run
// as two concurrent branches of the graph and join before the gradient
// assembly.
// CCB_SERIAL=1 runs every branch on the main stream in program order (the
// race check of tests/test_gpu_parity.py::test_branches_match_serial_order).
// graphs honour the per-node priorities captured from the branch streams
// (main = greatest, side / tail = least) instead of the launch stream's
static unsigned graph_flags() {
    static const unsigned f = [] {
        const char* e = std::getenv("CCB_NODE_PRIO");
        return (e && (e[0] == '1' || e[0] == '2')) ? unsigned(cudaGraphInstantiateFlagUseNodePriority) : 0u;
    }();
    return f;
}

static bool node_priorities() { return graph_flags() != 0u; }

// while capturing: the node(s) just added on `st` run at the least priority
void Trainer::note_low_priority(cudaStream_t st) {
    if (!node_priorities()) return;
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CCB_CUDA(cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd));
    if (cs != cudaStreamCaptureStatusActive) return;
    for (size_t i = 0; i < nd; ++i) low_nodes_.push_back(deps[i]);
}

// every other kernel node of a captured graph at the greatest priority, so
// the critical (distortion) chain's CTAs are dispatched before pending
// low-priority (ARM) CTAs whenever an SM frees up
void Trainer::apply_node_priorities(cudaGraph_t g) {
    if (!node_priorities()) return;
    int least = 0, greatest = 0;
    CCB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    size_t n = 0;
    CCB_CUDA(cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CCB_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
    for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType t;
        CCB_CUDA(cudaGraphNodeGetType(nd, &t));
        if (t != cudaGraphNodeTypeKernel) continue;
        const bool low = std::find(low_nodes_.begin(), low_nodes_.end(), nd) != low_nodes_.end();
        cudaKernelNodeAttrValue v{};
        static const bool invert = [] {  // CCB_NODE_PRIO=2: the ARM first instead
            const char* e = std::getenv("CCB_NODE_PRIO");
            return e && e[0] == '2';
        }();
        v.priority = (low != invert) ? least : greatest;
        CCB_CUDA(cudaGraphKernelNodeSetAttribute(nd, cudaLaunchAttributePriority, &v));
    }
    low_nodes_.clear();
}

static bool serial_branches() {
    static const bool on = [] {
        const char* e = std::getenv("CCB_SERIAL");
        return e && e[0] == '1';
    }();
    return on;
}
cudaStream_t Trainer::branch(bool tail) const {
    return serial_branches() ? stream_ : (tail ? tail_stream_ : side_stream_);
}
void Trainer::fork(bool tail) {
    if (serial_branches()) return;
    CCB_CUDA(cudaEventRecord(ev_fork_, stream_));
    CCB_CUDA(cudaStreamWaitEvent(branch(tail), ev_fork_, 0));
}
void Trainer::join(bool tail) {
    if (serial_branches()) return;
    CCB_CUDA(cudaEventRecord(ev_join_, branch(tail)));
    CCB_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
}
LaunchCtx Trainer::side(bool tail) const {
    LaunchCtx s = L_;
    s.stream = branch(tail);
    return s;
}

// timeline diagnostics (ccb_timeline): event marks inside the captured sequence
void Trainer::mark(int id, int on) {
    if (tl_ev_)  // an event-record node of the graph (timing), not a capture dependency
        CCB_CUDA(cudaEventRecordWithFlags(tl_ev_[id], on ? branch(on == 2) : stream_, cudaEventRecordExternal));
}

void Trainer::enqueue_proxy(bool batched) {
    mark(0, false);
    if (batched) launch_sched_load(L_);
    // constant-bank ARM: the weights packed into its constant slot on the
    // rate branch while the soft-quantiser runs
    fork();
    const bool prepped = launch_arm_prep(side());
    launch_softq_fwd(L_);
    mark(1, false);
    // A/B: the synthesis trunk's weight gradients as a separate launch on the
    // rate branch (1: after the dF pyramid, 2: before it) instead of fused
    // into the critical-chain backward (0).  Measured at 512x768: 0.483 ms
    // fused, 0.496 / 0.499 split — the recomputed hidden layer costs more than
    // the shorter critical chain saves.
    static const int mode = [] {
        const char* e = std::getenv("CCB_TRUNKW");
        return e ? std::atoi(e) : 0;
    }();
    fork();
    {
        LaunchCtx rate = side();
        rate.arm_prepped = prepped;
        launch_arm(rate, kArmProxy);
    }
    note_low_priority(side().stream);
    mark(2, true);
    if (mode != 2) {
        launch_pyramid(side());
        mark(3, true);
        CCB_CUDA(cudaEventRecord(ev_rate_, branch(false)));
    }
    launch_ups_forward(L_);
    mark(4, false);
    launch_syn_forward(L_, true);
    mark(5, false);
    if (mode == 0) {
        launch_syn_backward(L_, 0);
    } else {
        CCB_CUDA(cudaEventRecord(ev_synfwd_, stream_));
        CCB_CUDA(cudaStreamWaitEvent(branch(false), ev_synfwd_, 0));
        launch_syn_backward(side(), 2);
        launch_syn_backward(L_, 1);
    }
    if (mode == 2) {
        launch_pyramid(side());
        mark(3, true);
        CCB_CUDA(cudaEventRecord(ev_rate_, branch(false)));
    }
    mark(6, false);
    launch_ups_backward(L_, true, 0, 1);
    mark(7, false);
    // the remaining upsampling-backward stages do not read the rate branch;
    // the branches that do wait for it themselves (side: its own stream; tail:
    // below; main: before the coarse-grid gather)
    // The two finest grids (main levels 1, 0: ~93 % of the latents) have all
    // their gradient terms once the first upsampling-backward stage is done:
    // their gather and Adam step run beside the remaining (latency-bound)
    // coarse upsampling-backward stages.  The NN Adam step waits for every
    // gather (they read the IFCE weights).
    const int fine = H_.L >= 2 ? H_.main_gi[1] : 0;
    // NN gradients: every region but the upsampling taps is complete here
    // (ARM, synthesis); the taps ([off_tconv[0], off_c1w)) after the last stage
    const int ups_lo = H_.off_tconv[0], ups_hi = H_.off_c1w;
    // side (once the synthesis backward has written its partial rows): the
    // NN-gradient reductions that are complete; tail: cost / bias
    // corrections, the fine-grid gather and their Adam step
    fork();
    launch_nn_reduce(side(), 0, ups_lo);
    launch_nn_reduce(side(), ups_hi, H_.n_params);
    fork(true);
    if (!serial_branches()) CCB_CUDA(cudaStreamWaitEvent(branch(true), ev_rate_, 0));
    launch_finalize(side(true), kArmProxy, -1);
    launch_latent_grad_grids(side(true), fine, H_.n_grids);
    mark(8, 2);
    launch_adam_latents_grids(side(true), fine, H_.n_grids);
    launch_noise_ahead(side(true));  // next iteration's noise, in the tail's slack
    mark(9, 2);
    launch_ups_backward(L_, true, 1);
    mark(10, false);
    fork();  // the upsampling-tap reduction beside the coarse-grid gather
    launch_nn_reduce(side(), ups_lo, ups_hi);
    CCB_CUDA(cudaStreamWaitEvent(stream_, ev_rate_, 0));
    launch_latent_grad_grids(L_, 0, fine);
    mark(11, false);
    // every gather has read the weights: the NN step (side, after its
    // reductions) beside the coarse grids' Adam step (main)
    join(true);
    fork();
    nn_apply(side(), true, true, batched);
    if (fine > 0) launch_adam_latents_grids(L_, 0, fine);
    join();
    mark(12, false);
}

// Mean event times (ms after the iteration start) of the marks above over n
// graph replays of an instrumented proxy iteration.
void Trainer::timeline(int n, double lr, double temp, double noise, double* ms) {
    require_loaded();
    CCB_CUDA(cudaSetDevice(device_));
    h_scal_->lr = lr;
    h_scal_->temp = temp;
    h_scal_->noise = noise;
    CCB_CUDA(cudaMemcpyAsync(&H_.scal->lr, &h_scal_->lr, 3 * sizeof(double), cudaMemcpyHostToDevice,
                             stream_));
    std::vector<cudaEvent_t> ev(kTimelineMarks);
    for (auto& e : ev) CCB_CUDA(cudaEventCreate(&e));
    tl_ev_ = ev.data();
    cudaGraph_t g;
    CCB_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    enqueue_proxy(false);
    CCB_CUDA(cudaStreamEndCapture(stream_, &g));
    tl_ev_ = nullptr;
    cudaGraphExec_t ex;
    apply_node_priorities(g);
        CCB_CUDA(cudaGraphInstantiate(&ex, g, graph_flags()));
    cudaGraphDestroy(g);
    std::vector<double> acc(kTimelineMarks, 0.0);
    for (int it = 0; it < n; ++it) {
        CCB_CUDA(cudaGraphLaunch(ex, stream_));
        synchronize();
        for (int k = 1; k < kTimelineMarks; ++k) {
            float t = 0.0f;
            CCB_CUDA(cudaEventElapsedTime(&t, ev[0], ev[size_t(k)]));
            acc[size_t(k)] += t;
        }
    }
    cudaGraphExecDestroy(ex);
    for (auto& e : ev) cudaEventDestroy(e);
    for (int k = 0; k < kTimelineMarks; ++k) ms[k] = n > 0 ? acc[size_t(k)] / n : 0.0;
}

// Trainer::hardround_iteration (encoder.hpp:141-155)
void Trainer::enqueue_hardround(int slot) {
    fork();
    launch_arm(side(), kArmHard);
    launch_ups_forward(L_);
    launch_syn_forward(L_, true);
    launch_syn_backward(L_);
    launch_ups_backward(L_, false);
    join();
    launch_finalize(L_, kArmHard, slot);
    CCB_CUDA(cudaMemsetAsync(H_.lat_g, 0, sizeof(float) * size_t(H_.n_latents), stream_));
    if (slot >= 0) launch_snapshot_if_better(L_, slot, snaps_.at(slot).y, snaps_.at(slot).p);
    launch_nn_reduce(L_);
    nn_apply(L_, true, true, false);
}

// Trainer::true_cost (encoder.hpp:158-168)
void Trainer::enqueue_true_cost() {
    launch_quantize(L_, 255);
    launch_pads_from_q(L_);
    fork();
    launch_arm(side(), kArmForward);
    launch_ups_forward(L_);
    launch_syn_forward(L_, false);
    join();
    launch_finalize(L_, kArmForward, -1);
}

cudaGraphExec_t Trainer::ensure_graph(int which, int slot) {
    const int key = which == 3 ? 100 + slot : which;
    auto it = graphs_.find(key);
    if (it == graphs_.end()) {
        cudaGraph_t g;
        CCB_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
        if (which == 0) enqueue_proxy(false);
        else if (which == 1) enqueue_proxy(true);
        else if (which == 2) enqueue_true_cost();
        else enqueue_hardround(slot);
        CCB_CUDA(cudaStreamEndCapture(stream_, &g));
        cudaGraphExec_t ex;
        apply_node_priorities(g);
        CCB_CUDA(cudaGraphInstantiate(&ex, g, graph_flags()));
        cudaGraphDestroy(g);
        it = graphs_.emplace(key, ex).first;
    }
    return it->second;
}

void Trainer::run_graph(int which, int slot) {
    CCB_CUDA(cudaGraphLaunch(ensure_graph(which, slot), stream_));
}

void Trainer::read_scalars() {
    CCB_CUDA(cudaMemcpyAsync(h_scal_, H_.scal, sizeof(DevScalars), cudaMemcpyDeviceToHost, stream_));
    synchronize();
}

double Trainer::proxy_iteration(double lr, double temp, double noise_std) {
    require_loaded();
    CCB_CUDA(cudaSetDevice(device_));
    h_scal_->lr = lr;
    h_scal_->temp = temp;
    h_scal_->noise = noise_std;
    CCB_CUDA(cudaMemcpyAsync(&H_.scal->lr, &h_scal_->lr, 3 * sizeof(double),
                             cudaMemcpyHostToDevice, stream_));
    CCB_CUDA(cudaMemsetAsync(&H_.scal->halt, 0, sizeof(int), stream_));
    run_graph(0);
    read_scalars();
    last_mse_ = h_scal_->mse;
    last_bits_ = h_scal_->bits;
    return h_scal_->cost;
}

// ---------------------------------------------------------------- row bands
// One proxy iteration of a band is split around the exchange steps the band
// driver performs between ranks: (A) forward + backward up to
// local partial gradients; exchange halo-row latent gradients, NN-gradient
// partial sums and the bits / squared-error sums; (B) finish the gradients
// and the cost; AND the per-grid finiteness over ranks; (C) the Adam steps.
void Trainer::band_forward_backward(double lr, double temp, double noise_std, double* bits,
                                    double* se) {
    require_loaded();
    if (!band_.on) throw StateError("not a band trainer");
    CCB_CUDA(cudaSetDevice(device_));
    h_scal_->lr = lr;
    h_scal_->temp = temp;
    h_scal_->noise = noise_std;
    CCB_CUDA(cudaMemcpyAsync(&H_.scal->lr, &h_scal_->lr, 3 * sizeof(double),
                             cudaMemcpyHostToDevice, stream_));
    launch_softq_fwd(L_);
    fork();  // rate branch beside the distortion branch, as in enqueue_proxy
    launch_arm(side(), kArmProxy);
    launch_pyramid(side());
    launch_ups_forward(L_);
    launch_syn_forward(L_, true);
    launch_syn_backward(L_);
    launch_ups_backward(L_, true);
    join();
    launch_finalize(L_, kArmProxy, -1);  // local sums; latent grads are kept even if
    launch_latent_grad_partial(L_);      // this band's partial cost is not finite
    launch_nn_reduce(L_);
    read_scalars();
    *bits = h_scal_->bits;
    *se = h_scal_->mse * double(3 * H_.npix_global);
}

void Trainer::band_nn_partial(double* out) {
    CCB_CUDA(cudaMemcpyAsync(out, H_.grads_d, sizeof(double) * size_t(H_.n_params),
                             cudaMemcpyDeviceToHost, stream_));
    synchronize();
}

double Trainer::band_finish(const double* nn_sums, double bits, double se, int* lat_ok_own) {
    const int np = H_.n_params;
    std::vector<float> g(static_cast<size_t>(np));
    std::vector<int> ok(static_cast<size_t>(H_.n_tensors), 1);
    for (int p = 0; p < np; ++p) g[size_t(p)] = float(nn_sums[p]);
    for (int t = 0; t < H_.n_tensors; ++t)
        for (int e = 0; e < H_.tensor_size[t]; ++e)
            if (!std::isfinite(g[size_t(H_.tensor_off[t] + e)])) ok[size_t(t)] = 0;
    CCB_CUDA(cudaMemcpyAsync(H_.grads, g.data(), sizeof(float) * g.size(), cudaMemcpyHostToDevice,
                             stream_));
    CCB_CUDA(cudaMemcpyAsync(H_.tensor_ok, ok.data(), sizeof(int) * ok.size(),
                             cudaMemcpyHostToDevice, stream_));
    const double mse = se / double(3 * H_.npix_global);
    const double cost = std::fma(H_.lambda, bits / double(H_.npix_global), mse);  // encoder.hpp:115, as k_finalize
    h_scal_->bits = bits;
    h_scal_->mse = mse;
    h_scal_->cost = cost;
    h_scal_->cost_ok = std::isfinite(cost) ? 1 : 0;
    CCB_CUDA(cudaMemcpyAsync(&H_.scal->cost, &h_scal_->cost, 3 * sizeof(double),
                             cudaMemcpyHostToDevice, stream_));
    CCB_CUDA(cudaMemcpyAsync(&H_.scal->cost_ok, &h_scal_->cost_ok, sizeof(int),
                             cudaMemcpyHostToDevice, stream_));
    CCB_CUDA(cudaMemsetAsync(&H_.scal->halt, 0, sizeof(int), stream_));  // bands: the global cost decides
    launch_band_own_finite(L_);
    std::vector<int> lo(kMaxGrids);
    CCB_CUDA(cudaMemcpyAsync(lo.data(), H_.lat_ok, sizeof(int) * kMaxGrids, cudaMemcpyDeviceToHost,
                             stream_));
    synchronize();
    for (int gi = 0; gi < H_.n_grids; ++gi) lat_ok_own[gi] = lo[size_t(gi)];
    last_mse_ = mse;
    last_bits_ = bits;
    return cost;
}

// Device-resident band iteration: the schedule entry, the forward/backward
// and the step read everything from device memory, so a whole run of
// iterations is enqueued without host synchronisation (BandGroup, cc_band.cu).
void Trainer::band_reserve(int n) {
    require_loaded();
    if (!band_.on) throw StateError("not a band trainer");
    reserve_iterations(n);  // band trainers: buffers only, no iteration graph
}

void Trainer::band_dev_forward_backward() {
    require_loaded();
    if (!band_.on) throw StateError("not a band trainer");
    if (sched_cap_ <= 0) throw StateError("band_reserve before the device-resident band iteration");
    CCB_CUDA(cudaSetDevice(device_));
    launch_sched_load(L_);
    launch_softq_fwd(L_);
    fork();
    launch_arm(side(), kArmProxy);
    launch_pyramid(side());
    launch_ups_forward(L_);
    launch_syn_forward(L_, true);
    launch_syn_backward(L_);
    launch_ups_backward(L_, true);
    join();
    launch_finalize(L_, kArmProxy, -1);
    launch_latent_grad_partial(L_);
    launch_nn_reduce(L_);
    CCB_CUDA(cudaGetLastError());
}

void Trainer::band_dev_step() {
    CCB_CUDA(cudaSetDevice(device_));
    launch_adam_latents(L_);
    nn_apply(L_, true, true, true);  // + the iteration's record, sched_pos += 1
    CCB_CUDA(cudaGetLastError());
}

void Trainer::band_step(const int* lat_ok) {
    CCB_CUDA(cudaMemcpyAsync(H_.lat_ok, lat_ok, sizeof(int) * size_t(H_.n_grids),
                             cudaMemcpyHostToDevice, stream_));
    launch_adam_latents(L_);
    nn_apply(L_, true, true, false);
    read_scalars();
}

// Global rows [rb, re) of grid gi, flat (rows x cols): mode 0 get, 1 set, 2 add.
void Trainer::band_rows(int which, int gi, int rb, int re, float* buf, int mode) {
    if (gi < 0 || gi >= H_.n_grids) throw ConfigError("grid index out of range");
    const GridGeom& g = H_.g[gi];
    if (rb < g.row0 || re > g.row0 + g.rows || rb > re) throw ConfigError("rows outside the band window");
    float* base = (which == 0 ? H_.y : which == 1 ? H_.lat_g : nullptr);
    if (!base) throw ConfigError("band_rows: which must be 0 (latents) or 1 (latent grads)");
    float* d = base + g.lat_off + int64_t(rb - g.row0) * g.cols;
    const size_t n = size_t(re - rb) * size_t(g.cols);
    if (n == 0) return;
    if (mode == 0) {
        CCB_CUDA(cudaMemcpyAsync(buf, d, sizeof(float) * n, cudaMemcpyDeviceToHost, stream_));
    } else if (mode == 1) {
        CCB_CUDA(cudaMemcpyAsync(d, buf, sizeof(float) * n, cudaMemcpyHostToDevice, stream_));
    } else {
        std::vector<float> cur(n);
        CCB_CUDA(cudaMemcpyAsync(cur.data(), d, sizeof(float) * n, cudaMemcpyDeviceToHost, stream_));
        synchronize();
        for (size_t i = 0; i < n; ++i) cur[i] += buf[i];
        CCB_CUDA(cudaMemcpyAsync(d, cur.data(), sizeof(float) * n, cudaMemcpyHostToDevice, stream_));
    }
    synchronize();
}

void* Trainer::band_device_rows(int which, int gi, int rb, int re, int64_t* count) {
    if (gi < 0 || gi >= H_.n_grids) throw ConfigError("grid index out of range");
    const GridGeom& g = H_.g[gi];
    if (rb < g.row0 || re > g.row0 + g.rows || rb > re) throw ConfigError("rows outside the band window");
    float* base = (which == 0 ? H_.y : which == 1 ? H_.lat_g : nullptr);
    if (!base) throw ConfigError("which must be 0 (latents) or 1 (latent grads)");
    *count = int64_t(re - rb) * g.cols;
    return base + g.lat_off + int64_t(rb - g.row0) * g.cols;
}

void Trainer::band_grid_rows(int gi, int* out4) const {
    const GridGeom& g = H_.g[gi];
    out4[0] = g.row0;
    out4[1] = g.row0 + g.own_lo;
    out4[2] = g.row0 + g.own_hi;
    out4[3] = g.row0 + g.rows;
}

void Trainer::proxy_iterations(int n, const double* lr, const double* temp, const double* noise,
                               double* rec) {
    enqueue_proxy_iterations(n, lr, temp, noise);
    if (n <= 0) return;
    std::vector<double> r(4 * size_t(n));
    last_records(n, r.data());
    if (rec) std::memcpy(rec, r.data(), sizeof(double) * r.size());
}

void Trainer::last_records(int n, double* rec) {
    if (n <= 0) return;
    if (n > sched_cap_) throw ConfigError("more records requested than the last batch holds");
    read_scalars();  // synchronises the stream: the kernels' host writes have landed
    std::memcpy(rec, h_rec_, sizeof(double) * 4 * size_t(n));
    last_mse_ = rec[4 * size_t(n - 1) + 1];
    last_bits_ = rec[4 * size_t(n - 1) + 2];
}

void Trainer::set_stream(cudaStream_t s) {
    synchronize();
    stream_ = s ? s : own_stream_;
    L_.stream = stream_;
}

void Trainer::reserve_iterations(int n) {
    require_loaded();
    CCB_CUDA(cudaSetDevice(device_));
    if (n > sched_cap_) {
        synchronize();
        if (d_sched_) cudaFree(d_sched_);
        CCB_CUDA(cudaMalloc(&d_sched_, sizeof(double) * 3 * size_t(n)));
        // the records live in mapped pinned host memory: k_nn_step writes each
        // iteration's record straight to the host (no copy between graphs)
        if (h_rec_) cudaFreeHost(h_rec_);
        CCB_CUDA(cudaHostAlloc(&h_rec_, sizeof(double) * 4 * size_t(n), cudaHostAllocMapped));
        CCB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_rec_), h_rec_, 0));
        if (h_sched_) cudaFreeHost(h_sched_);
        CCB_CUDA(cudaMallocHost(&h_sched_, sizeof(double) * 3 * size_t(n)));
        sched_cap_ = n;
        H_.sched = d_sched_;  // read by k_sched_load / k_nn_step through the plan
        H_.rec = d_rec_;
        CCB_CUDA(cudaMemcpy(d_plan_, &H_, sizeof(Plan), cudaMemcpyHostToDevice));
        auto it = graphs_.find(1);  // (captured before the buffers moved)
        if (it != graphs_.end()) {
            cudaGraphExecDestroy(it->second);
            graphs_.erase(it);
        }
    }
    if (!band_.on) ensure_graph(1);
}

void Trainer::enqueue_proxy_iterations(int n, const double* lr, const double* temp,
                                       const double* noise) {
    require_loaded();
    if (n <= 0) return;
    reserve_iterations(n);  // no-op once sized: buffers and the graph are reused
    upload_schedule(n, lr, temp, noise);  // from pinned memory
    reset_batch_counters();
    // every iteration's record (cost, mse, bits, global_iter) is written by
    // the iteration's last kernel into mapped pinned host memory, without a
    // host synchronisation or a copy between the graphs
    for (int i = 0; i < n; ++i) run_graph(1);
}

void Trainer::upload_schedule(int n, const double* lr, const double* temp, const double* noise) {
    if (cudaEventQuery(ev_sched_) != cudaSuccess) {  // the previous batch's upload has left h_sched_
        count_host_sync();
        CCB_CUDA(cudaEventSynchronize(ev_sched_));
    }
    for (int i = 0; i < n; ++i) {
        h_sched_[3 * i] = lr[i];
        h_sched_[3 * i + 1] = temp[i];
        h_sched_[3 * i + 2] = noise[i];
    }
    CCB_CUDA(cudaMemcpyAsync(d_sched_, h_sched_, sizeof(double) * 3 * size_t(n), cudaMemcpyHostToDevice,
                             stream_));
    CCB_CUDA(cudaEventRecord(ev_sched_, stream_));
}

void Trainer::reset_batch_counters() {
    CCB_CUDA(cudaMemsetAsync(&H_.scal->sched_pos, 0, sizeof(int64_t), stream_));
    CCB_CUDA(cudaMemsetAsync(&H_.scal->halt, 0, sizeof(int), stream_));
}

cudaGraphExec_t Trainer::capture_batched_proxy(const Plan* d_plans, int batch, float* const* arm_cstages) {
    const LaunchCtx keep = L_;
    L_.plan = d_plans;
    L_.batch = batch;
    L_.arm_cstages = arm_cstages;
    cudaGraph_t g;
    cudaGraphExec_t ex = nullptr;
    try {
        CCB_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
        enqueue_proxy(true);
        CCB_CUDA(cudaStreamEndCapture(stream_, &g));
        apply_node_priorities(g);
        CCB_CUDA(cudaGraphInstantiate(&ex, g, graph_flags()));
        cudaGraphDestroy(g);
    } catch (...) {
        L_ = keep;
        throw;
    }
    L_ = keep;
    return ex;
}

Batch::Batch(std::vector<Trainer*> trainers) : t_(std::move(trainers)) {
    if (t_.empty()) throw ConfigError("empty batch");
    const Plan& a = t_[0]->host_plan();
    for (Trainer* t : t_) {
        const Plan& b = t->host_plan();
        if (t->is_band()) throw ConfigError("row-band trainers cannot be batched");
        if (b.H != a.H || b.W != a.W || b.n_latents != a.n_latents || b.n_params != a.n_params ||
            b.D != a.D || b.Wd != a.Wd || b.syn_F != a.syn_F || b.posts != a.posts || b.use_soap != a.use_soap ||
            b.n_grids != a.n_grids)
            throw ConfigError("batched trainers must share the image size, decoder and optimizer");
        t->set_stream(t_[0]->stream());
    }
}

Batch::~Batch() {
    if (graph_) cudaGraphExecDestroy(graph_);
    if (d_plans_) cudaFree(d_plans_);
    // every trainer back on its own stream (they were moved onto trainers[0]'s)
    for (size_t b = 1; b < t_.size(); ++b) {
        try {
            t_[b]->set_stream(nullptr);
        } catch (...) {
        }
    }
}

void Batch::reserve_iterations(int n) {
    if (n <= cap_ && graph_) return;
    for (Trainer* t : t_) t->reserve_iterations(n);
    if (graph_) {
        cudaGraphExecDestroy(graph_);
        graph_ = nullptr;
    }
    const size_t B = t_.size();
    std::vector<Plan> hp(B);
    for (size_t b = 0; b < B; ++b) {
        hp[b] = t_[b]->host_plan();
        hp[b].sched = t_[0]->device_schedule();  // one schedule for the whole batch
    }
    if (!d_plans_) CCB_CUDA(cudaMalloc(&d_plans_, sizeof(Plan) * B));
    CCB_CUDA(cudaMemcpy(d_plans_, hp.data(), sizeof(Plan) * B, cudaMemcpyHostToDevice));
    stages_.resize(B);
    for (size_t b = 0; b < B; ++b) stages_[b] = hp[b].arm_cstage;
    graph_ = t_[0]->capture_batched_proxy(d_plans_, int(B), stages_.data());
    cap_ = n;
}

void Batch::enqueue_proxy_iterations(int n, const double* lr, const double* temp, const double* noise) {
    if (n <= 0) return;
    reserve_iterations(n);
    t_[0]->upload_schedule(n, lr, temp, noise);
    for (Trainer* t : t_) t->reset_batch_counters();
    for (int i = 0; i < n; ++i) CCB_CUDA(cudaGraphLaunch(graph_, t_[0]->stream()));
}

void Batch::synchronize() {
    count_host_sync();
    CCB_CUDA(cudaStreamSynchronize(t_[0]->stream()));
}

// Stage-by-stage replay of one proxy iteration with events in between
// (diagnostics; same kernels as the graph).
void Trainer::profile_stages(int n, double lr, double temp, double noise, double* ms) {
    require_loaded();
    CCB_CUDA(cudaSetDevice(device_));
    h_scal_->lr = lr;
    h_scal_->temp = temp;
    h_scal_->noise = noise;
    CCB_CUDA(cudaMemcpyAsync(&H_.scal->lr, &h_scal_->lr, 3 * sizeof(double),
                             cudaMemcpyHostToDevice, stream_));
    constexpr int NS = 8;
    cudaEvent_t ev[NS + 1];
    for (auto& e : ev) CCB_CUDA(cudaEventCreate(&e));
    double acc[NS] = {0};
    for (int it = 0; it < n; ++it) {
        CCB_CUDA(cudaEventRecord(ev[0], stream_));
        launch_softq_fwd(L_);
        CCB_CUDA(cudaEventRecord(ev[1], stream_));
        launch_arm(L_, kArmProxy);
        CCB_CUDA(cudaEventRecord(ev[2], stream_));
        launch_pyramid(L_);
        CCB_CUDA(cudaEventRecord(ev[3], stream_));
        launch_ups_forward(L_);
        CCB_CUDA(cudaEventRecord(ev[4], stream_));
        launch_syn_forward(L_, true);
        CCB_CUDA(cudaEventRecord(ev[5], stream_));
        launch_syn_backward(L_);
        CCB_CUDA(cudaEventRecord(ev[6], stream_));
        launch_ups_backward(L_, true);
        CCB_CUDA(cudaEventRecord(ev[7], stream_));
        launch_finalize(L_, kArmProxy, -1);
        launch_latent_grad(L_);
        launch_adam_latents(L_);
        launch_nn_reduce(L_);
        nn_apply(L_, true, true, false);
        CCB_CUDA(cudaEventRecord(ev[8], stream_));
        CCB_CUDA(cudaEventSynchronize(ev[8]));
        for (int s = 0; s < NS; ++s) {
            float t = 0.f;
            CCB_CUDA(cudaEventElapsedTime(&t, ev[s], ev[s + 1]));
            acc[s] += t;
        }
    }
    for (int s = 0; s < NS; ++s) ms[s] = acc[s] / std::max(1, n);
    for (auto& e : ev) cudaEventDestroy(e);
}

// Kernel nodes of one batched proxy iteration (the graph the benchmark and
// cc_trainer_train replay; the schedule-load kernel included).
int Trainer::kernels_per_iteration() {
    cudaGraph_t g;
    CCB_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    enqueue_proxy(true);
    CCB_CUDA(cudaStreamEndCapture(stream_, &g));
    size_t n = 0;
    CCB_CUDA(cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CCB_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
    int k = 0;
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        CCB_CUDA(cudaGraphNodeGetType(nd, &t));
        if (t == cudaGraphNodeTypeKernel) ++k;
    }
    cudaGraphDestroy(g);
    return k;
}

void Trainer::ensure_snapshot(int slot) {
    if (slot < 0 || slot >= kSnapSlots) throw ConfigError("snapshot slot must be in [0, 8)");
    if (snaps_.count(slot)) return;
    SnapSlot s;
    CCB_CUDA(cudaMalloc(&s.y, sizeof(float) * size_t(H_.n_latents)));
    CCB_CUDA(cudaMalloc(&s.p, sizeof(float) * size_t(H_.n_params)));
    s.valid = false;
    snaps_[slot] = s;
    const double inf = std::numeric_limits<double>::infinity();
    h_scal_->snap_cost[slot] = inf;
    CCB_CUDA(cudaMemcpyAsync(&H_.scal->snap_cost[slot], &h_scal_->snap_cost[slot], sizeof(double),
                             cudaMemcpyHostToDevice, stream_));
    synchronize();
}

double Trainer::hardround_iteration(double lr, int best_slot) {
    require_loaded();
    CCB_CUDA(cudaSetDevice(device_));
    if (best_slot >= 0) ensure_snapshot(best_slot);
    h_scal_->lr = lr;
    CCB_CUDA(cudaMemcpyAsync(&H_.scal->lr, &h_scal_->lr, sizeof(double), cudaMemcpyHostToDevice,
                             stream_));
    run_graph(3, best_slot);
    read_scalars();
    last_mse_ = h_scal_->mse;
    last_bits_ = h_scal_->bits;
    if (best_slot >= 0 && h_scal_->snap_take) snaps_[best_slot].valid = true;
    return h_scal_->cost;
}

double Trainer::true_cost(double* psnr, double* bpp) {
    require_loaded();
    CCB_CUDA(cudaSetDevice(device_));
    run_graph(2);
    read_scalars();
    const double mse = h_scal_->mse, bits = h_scal_->bits;
    if (psnr) *psnr = mse > 0 ? std::min(99.0, -10.0 * std::log10(mse)) : 99.0;  // kPsnrCap
    if (bpp) *bpp = bits / double(H_.npix);
    return h_scal_->cost;
}

void Trainer::quantize_all() {
    require_loaded();
    launch_quantize(L_, 255);
    synchronize();
}

void Trainer::load_pads_from_q() {
    require_loaded();
    launch_pads_from_q(L_);
    synchronize();
}

void Trainer::snapshot(int slot, double cost) {
    require_loaded();
    ensure_snapshot(slot);
    SnapSlot& s = snaps_[slot];
    CCB_CUDA(cudaMemcpyAsync(s.y, H_.y, sizeof(float) * size_t(H_.n_latents),
                             cudaMemcpyDeviceToDevice, stream_));
    CCB_CUDA(cudaMemcpyAsync(s.p, H_.params, sizeof(float) * size_t(H_.n_params),
                             cudaMemcpyDeviceToDevice, stream_));
    h_scal_->snap_cost[slot] = cost;
    CCB_CUDA(cudaMemcpyAsync(&H_.scal->snap_cost[slot], &h_scal_->snap_cost[slot], sizeof(double),
                             cudaMemcpyHostToDevice, stream_));
    s.valid = true;
    synchronize();
}

double Trainer::snapshot_cost(int slot) {
    if (!snaps_.count(slot)) return std::numeric_limits<double>::infinity();
    read_scalars();
    return h_scal_->snap_cost[slot];
}

void Trainer::restore(int slot) {
    require_loaded();
    auto it = snaps_.find(slot);
    if (it == snaps_.end() || !it->second.valid) throw StateError("empty snapshot slot");
    CCB_CUDA(cudaMemcpyAsync(H_.y, it->second.y, sizeof(float) * size_t(H_.n_latents),
                             cudaMemcpyDeviceToDevice, stream_));
    CCB_CUDA(cudaMemcpyAsync(H_.params, it->second.p, sizeof(float) * size_t(H_.n_params),
                             cudaMemcpyDeviceToDevice, stream_));
    synchronize();
}

void Trainer::take_candidate(int slot, double cost) {
    require_loaded();
    CandSlot& c = cands_[slot];
    const size_t nl = size_t(H_.n_latents), np = size_t(H_.n_params);
    if (!c.y) {
        CCB_CUDA(cudaMalloc(&c.y, sizeof(float) * nl));
        CCB_CUDA(cudaMalloc(&c.m, sizeof(float) * nl));
        CCB_CUDA(cudaMalloc(&c.v, sizeof(float) * nl));
        CCB_CUDA(cudaMalloc(&c.p, sizeof(float) * np));
        CCB_CUDA(cudaMalloc(&c.nm, sizeof(float) * np));
        CCB_CUDA(cudaMalloc(&c.nv, sizeof(float) * np));
        if (H_.use_soap) CCB_CUDA(cudaMalloc(&c.soap, sizeof(double) * size_t(sizes_.soap)));
    }
    auto cp = [&](void* d, const void* s, size_t b) {
        CCB_CUDA(cudaMemcpyAsync(d, s, b, cudaMemcpyDeviceToDevice, stream_));
    };
    cp(c.y, H_.y, sizeof(float) * nl);
    cp(c.m, H_.lat_m, sizeof(float) * nl);
    cp(c.v, H_.lat_v, sizeof(float) * nl);
    cp(c.p, H_.params, sizeof(float) * np);
    cp(c.nm, H_.nn_m, sizeof(float) * np);
    cp(c.nv, H_.nn_v, sizeof(float) * np);
    if (H_.use_soap) cp(c.soap, H_.soap, sizeof(double) * size_t(sizes_.soap));
    c.lat_t.resize(kMaxGrids);
    c.nn_t.resize(kMaxTensors);
    CCB_CUDA(cudaMemcpyAsync(c.lat_t.data(), H_.lat_t, sizeof(int64_t) * kMaxGrids,
                             cudaMemcpyDeviceToHost, stream_));
    CCB_CUDA(cudaMemcpyAsync(c.nn_t.data(), H_.nn_t, sizeof(int64_t) * kMaxTensors,
                             cudaMemcpyDeviceToHost, stream_));
    c.cost = cost;
    synchronize();
    loaded_ = false;
}

void Trainer::load_candidate(int slot) {
    auto it = cands_.find(slot);
    if (it == cands_.end()) throw StateError("empty candidate slot");
    CandSlot& c = it->second;
    const size_t nl = size_t(H_.n_latents), np = size_t(H_.n_params);
    auto cp = [&](void* d, const void* s, size_t b) {
        CCB_CUDA(cudaMemcpyAsync(d, s, b, cudaMemcpyDeviceToDevice, stream_));
    };
    cp(H_.y, c.y, sizeof(float) * nl);
    cp(H_.lat_m, c.m, sizeof(float) * nl);
    cp(H_.lat_v, c.v, sizeof(float) * nl);
    cp(H_.params, c.p, sizeof(float) * np);
    cp(H_.nn_m, c.nm, sizeof(float) * np);
    cp(H_.nn_v, c.nv, sizeof(float) * np);
    if (H_.use_soap) cp(H_.soap, c.soap, sizeof(double) * size_t(sizes_.soap));
    CCB_CUDA(cudaMemcpyAsync(H_.lat_t, c.lat_t.data(), sizeof(int64_t) * kMaxGrids,
                             cudaMemcpyHostToDevice, stream_));
    CCB_CUDA(cudaMemcpyAsync(H_.nn_t, c.nn_t.data(), sizeof(int64_t) * kMaxTensors,
                             cudaMemcpyHostToDevice, stream_));
    zero_pads();  // setup_buffers (encoder.hpp:217-235)
    synchronize();
    cur_cost_ = c.cost;
    for (float* p : {c.y, c.m, c.v, c.p, c.nm, c.nv}) cudaFree(p);
    if (c.soap) cudaFree(c.soap);
    cands_.erase(it);
    loaded_ = true;
}

void Trainer::discard_candidate(int slot) {
    auto it = cands_.find(slot);
    if (it == cands_.end()) return;
    CandSlot& c = it->second;
    synchronize();
    for (float* p : {c.y, c.m, c.v, c.p, c.nm, c.nv}) cudaFree(p);
    if (c.soap) cudaFree(c.soap);
    cands_.erase(it);
}

double Trainer::candidate_cost(int slot) const {
    auto it = cands_.find(slot);
    if (it == cands_.end()) throw StateError("empty candidate slot");
    return it->second.cost;
}

int64_t Trainer::global_iter() {
    read_scalars();
    return h_scal_->global_iter;
}

int Trainer::skipped_steps() {
    read_scalars();
    return h_scal_->skipped;
}

void Trainer::set_counters(int64_t gi, int skipped) {
    read_scalars();
    h_scal_->global_iter = gi;
    h_scal_->skipped = skipped;
    CCB_CUDA(cudaMemcpyAsync(H_.scal, h_scal_, sizeof(DevScalars), cudaMemcpyHostToDevice, stream_));
    synchronize();
}

void Trainer::set_state(const float* lat, const float* par, const float* lm, const float* lv,
                        const int64_t* lt, const float* nm, const float* nv, const int64_t* nt) {
    require_loaded();
    if (H_.use_soap && (nm || nv || nt))  // as the reference ABI (oracle/ref_capi.cpp)
        throw ConfigError("optimizer state transfer needs use_soap = false");
    const size_t nl = size_t(H_.n_latents), np = size_t(H_.n_params);
    auto up = [&](void* d, const void* s, size_t b) {
        if (s) CCB_CUDA(cudaMemcpyAsync(d, s, b, cudaMemcpyHostToDevice, stream_));
    };
    up(H_.y, lat, sizeof(float) * nl);
    up(H_.params, par, sizeof(float) * np);
    up(H_.lat_m, lm, sizeof(float) * nl);
    up(H_.lat_v, lv, sizeof(float) * nl);
    up(H_.lat_t, lt, sizeof(int64_t) * size_t(H_.n_grids));
    up(H_.nn_m, nm, sizeof(float) * np);
    up(H_.nn_v, nv, sizeof(float) * np);
    up(H_.nn_t, nt, sizeof(int64_t) * size_t(H_.n_tensors));
    synchronize();
}

void Trainer::get_state(float* lat, float* par, float* lm, float* lv, int64_t* lt, float* nm,
                        float* nv, int64_t* nt) {
    require_loaded();
    if (H_.use_soap && (nm || nv || nt))
        throw ConfigError("optimizer state transfer needs use_soap = false");
    const size_t nl = size_t(H_.n_latents), np = size_t(H_.n_params);
    auto dn = [&](void* d, const void* s, size_t b) {
        if (d) CCB_CUDA(cudaMemcpyAsync(d, s, b, cudaMemcpyDeviceToHost, stream_));
    };
    dn(lat, H_.y, sizeof(float) * nl);
    dn(par, H_.params, sizeof(float) * np);
    dn(lm, H_.lat_m, sizeof(float) * nl);
    dn(lv, H_.lat_v, sizeof(float) * nl);
    dn(lt, H_.lat_t, sizeof(int64_t) * size_t(H_.n_grids));
    dn(nm, H_.nn_m, sizeof(float) * np);
    dn(nv, H_.nn_v, sizeof(float) * np);
    dn(nt, H_.nn_t, sizeof(int64_t) * size_t(H_.n_tensors));
    synchronize();
}

// ---------------------------------------------------------------- decode passes
// encode_image's amplitude-clamped q (bitstream.hpp:194-197) -> device.
void Trainer::set_q(const int32_t* q) {
    require_loaded();
    CCB_CUDA(cudaMemcpyAsync(H_.q, q, sizeof(int32_t) * size_t(H_.n_latents), cudaMemcpyHostToDevice,
                             stream_));
    launch_pads_from_q(L_);
    synchronize();
}

// latent_rate_estimate / mse_rgb(reconstruct_image) (decode_core.hpp:38-63) on
// the current q with `params` substituted for the call.
void Trainer::decode_terms(const float* params, int which, double* bits, double* mse) {
    require_loaded();
    const size_t np = size_t(H_.n_params);
    if (params) {
        if (!d_param_save_) d_param_save_ = static_cast<float*>(dalloc(sizeof(float) * np));
        CCB_CUDA(cudaMemcpyAsync(d_param_save_, H_.params, sizeof(float) * np, cudaMemcpyDeviceToDevice,
                                 stream_));
        CCB_CUDA(cudaMemcpyAsync(H_.params, params, sizeof(float) * np, cudaMemcpyHostToDevice, stream_));
    }
    launch_pads_from_q(L_);
    if (which & 1) launch_arm(L_, kArmForward);
    if (which & 2) {
        launch_ups_forward(L_);
        launch_syn_forward(L_, false);
    }
    launch_finalize(L_, kArmForward, -1);
    if (params)
        CCB_CUDA(cudaMemcpyAsync(H_.params, d_param_save_, sizeof(float) * np, cudaMemcpyDeviceToDevice,
                                 stream_));
    read_scalars();
    if (bits && (which & 1)) *bits = h_scal_->bits;
    if (mse && (which & 2)) *mse = h_scal_->mse;
}

// encode_latents' per-latent (mu, sigma) (bitstream.hpp:106-141) on the device
void Trainer::latent_mu_sigma(const float* params, float* mu, float* sigma) {
    require_loaded();
    if (band_.on) throw ConfigError("latent entropy coding needs the whole image (not a row band)");
    const size_t np = size_t(H_.n_params), nl = size_t(H_.n_latents);
    if (params) {
        if (!d_param_save_) d_param_save_ = static_cast<float*>(dalloc(sizeof(float) * np));
        CCB_CUDA(cudaMemcpyAsync(d_param_save_, H_.params, sizeof(float) * np, cudaMemcpyDeviceToDevice,
                                 stream_));
        CCB_CUDA(cudaMemcpyAsync(H_.params, params, sizeof(float) * np, cudaMemcpyHostToDevice, stream_));
    }
    if (!d_mu_sigma_) d_mu_sigma_ = static_cast<float*>(dalloc(sizeof(float) * 2 * nl));
    launch_latent_mu_sigma(L_, d_mu_sigma_, d_mu_sigma_ + nl);
    if (params)
        CCB_CUDA(cudaMemcpyAsync(H_.params, d_param_save_, sizeof(float) * np, cudaMemcpyDeviceToDevice,
                                 stream_));
    if (mu) CCB_CUDA(cudaMemcpyAsync(mu, d_mu_sigma_, sizeof(float) * nl, cudaMemcpyDeviceToHost, stream_));
    if (sigma)
        CCB_CUDA(cudaMemcpyAsync(sigma, d_mu_sigma_ + nl, sizeof(float) * nl, cudaMemcpyDeviceToHost, stream_));
    synchronize();
}

void Trainer::soap_state(double* arena, float* m1, float* v2, int64_t* t, int64_t* n_arena) {
    require_loaded();
    if (!H_.use_soap) throw ConfigError("not a SOAP trainer (use_soap = false)");
    if (n_arena) *n_arena = sizes_.soap;
    const size_t np = size_t(H_.n_params);
    if (arena)
        CCB_CUDA(cudaMemcpyAsync(arena, H_.soap, sizeof(double) * size_t(sizes_.soap),
                                 cudaMemcpyDeviceToHost, stream_));
    if (m1) CCB_CUDA(cudaMemcpyAsync(m1, H_.nn_m, sizeof(float) * np, cudaMemcpyDeviceToHost, stream_));
    if (v2) CCB_CUDA(cudaMemcpyAsync(v2, H_.nn_v, sizeof(float) * np, cudaMemcpyDeviceToHost, stream_));
    if (t)
        CCB_CUDA(cudaMemcpyAsync(t, H_.nn_t, sizeof(int64_t) * size_t(H_.n_tensors),
                                 cudaMemcpyDeviceToHost, stream_));
    synchronize();
}

void Trainer::set_soap_state(const double* arena, const float* m1, const float* v2, const int64_t* t) {
    require_loaded();
    if (!H_.use_soap) throw ConfigError("not a SOAP trainer (use_soap = false)");
    const size_t np = size_t(H_.n_params);
    if (arena)
        CCB_CUDA(cudaMemcpyAsync(H_.soap, arena, sizeof(double) * size_t(sizes_.soap),
                                 cudaMemcpyHostToDevice, stream_));
    if (m1) CCB_CUDA(cudaMemcpyAsync(H_.nn_m, m1, sizeof(float) * np, cudaMemcpyHostToDevice, stream_));
    if (v2) CCB_CUDA(cudaMemcpyAsync(H_.nn_v, v2, sizeof(float) * np, cudaMemcpyHostToDevice, stream_));
    if (t)
        CCB_CUDA(cudaMemcpyAsync(H_.nn_t, t, sizeof(int64_t) * size_t(H_.n_tensors),
                                 cudaMemcpyHostToDevice, stream_));
    synchronize();
}

void Trainer::get_grads(float* lg, float* pg) {
    require_loaded();
    if (lg)
        CCB_CUDA(cudaMemcpyAsync(lg, H_.lat_g, sizeof(float) * size_t(H_.n_latents),
                                 cudaMemcpyDeviceToHost, stream_));
    if (pg)
        CCB_CUDA(cudaMemcpyAsync(pg, H_.grads, sizeof(float) * size_t(H_.n_params),
                                 cudaMemcpyDeviceToHost, stream_));
    synchronize();
}

void Trainer::get_q(int32_t* q) {
    require_loaded();
    CCB_CUDA(cudaMemcpyAsync(q, H_.q, sizeof(int32_t) * size_t(H_.n_latents), cudaMemcpyDeviceToHost,
                             stream_));
    synchronize();
}

void Trainer::get_params(float* p) {
    CCB_CUDA(cudaMemcpyAsync(p, H_.params, sizeof(float) * size_t(H_.n_params),
                             cudaMemcpyDeviceToHost, stream_));
    synchronize();
}

}  // namespace ccb
