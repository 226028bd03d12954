// cc_capi.cu — the extern "C" boundary (include/coolchic_b200.h) of the B200
// library, plus warmup / train: the reference's host-side schedule logic
// (encoder.hpp:315-413) re-hosted over the device-resident Trainer so the main
// stage runs in chunks of graph replays between true-cost evaluations.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <limits>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "../../include/coolchic_b200.h"
#include "../../include/coolchic_b200_diag.h"
#include "../../include/coolchic_synth.h"
#include "cc_band.h"
#include "cc_runtime.h"

using ccb::Trainer;

struct cc_batch {
    std::unique_ptr<ccb::Batch> b;
};
struct cc_band_group {
    std::unique_ptr<ccb::BandGroup> g;
};

struct cc_trainer {
    std::unique_ptr<Trainer> tr;
    std::vector<float> image;  // host copy (train() restarts from it)
    int h = 0, w = 0;
    cc_encoder_config enc{};
    cc_decoder_config dec{};
    std::string log_path;
    int device = 0;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const ccb::ConfigError& e) {
        return fail(CC_ERR_CONFIG, e.what());
    } catch (const ccb::CudaError& e) {
        return fail(CC_ERR_CUDA, e.what());
    } catch (const ccb::StateError& e) {
        return fail(CC_ERR_STATE, e.what());
    } catch (const std::exception& e) {
        return fail(CC_ERR_STATE, e.what());
    }
}

// Schedule::value (config.hpp:23-29)
double sched_value(double start, double end, bool cosine, int horizon, int iter) {
    if (iter <= 0) return start;
    if (iter >= horizon) return end;
    const double t = double(iter) / double(horizon);
    if (!cosine) return start + (end - start) * t;
    return end + (start - end) * (1.0 + std::cos(3.141592653589793 * t)) * 0.5;
}

cc_encoder_config default_enc() {
    cc_encoder_config c{};
    c.warmup_candidates = 5;
    c.warmup_keep = 2;
    c.warmup_iters = 400;
    c.main_iters = 96700;
    c.hardround_iters = 500;
    c.lr_start = 1e-2;
    c.lr_end = 1e-6;
    c.noise_std_start = 0.22;
    c.noise_std_end = 0.15;
    c.temp_start = 0.35;
    c.temp_end = 0.08;
    c.hardround_lr = 1e-4;
    c.lambda = 0.001;
    c.seed = 0;
    c.use_soap = 1;  // EncoderConfig{} (config.hpp:107); the benchmarks set 0
    c.true_cost_interval = 1000;
    c.log_path = nullptr;
    return c;
}

int warmup_total(const cc_encoder_config& c) { return (c.warmup_candidates + c.warmup_keep) * c.warmup_iters; }

// CSV log (encoder.hpp:201-207, 279-287)
struct Log {
    std::ofstream f;
    explicit Log(const std::string& path) {
        if (!path.empty()) {
            f.open(path);
            if (f) f << "iter,proxy_cost,true_cost,psnr,bpp\n";
        }
    }
    void row(int64_t gi, double proxy, const double* truec, double mse, double bits, double npix) {
        if (!f) return;
        const double psnr = mse > 0 ? -10.0 * std::log10(mse) : 99.0;
        f << gi << "," << proxy << ",";
        if (truec) f << *truec;
        f << "," << psnr << "," << bits / npix << "\n";
    }
    ~Log() {
        if (f) f.flush();
    }
};

// n proxy iterations at fixed scalars (warm-up)
void run_fixed(Trainer& tr, int n, double lr, double temp, double noise) {
    if (n <= 0) return;
    std::vector<double> a(n, lr), b(n, temp), c(n, noise);
    tr.proxy_iterations(n, a.data(), b.data(), c.data(), nullptr);
}

}  // namespace

namespace ccb {

namespace {

// One candidate's full trainer state (CandidateState, encoder.hpp:42-48) from
// one trainer into another of the same geometry.
void copy_candidate(Trainer& src, Trainer& dst) {
    const Plan& p = src.plan();
    const size_t nl = size_t(p.n_latents), np = size_t(p.n_params);
    std::vector<float> lat(nl), lm(nl), lv(nl), par(np), nm(np), nv(np);
    std::vector<int64_t> lt(static_cast<size_t>(p.n_grids)), nt(static_cast<size_t>(p.n_tensors));
    const bool soap = p.use_soap != 0;
    src.get_state(lat.data(), par.data(), lm.data(), lv.data(), lt.data(), soap ? nullptr : nm.data(),
                  soap ? nullptr : nv.data(), soap ? nullptr : nt.data());
    dst.set_state(lat.data(), par.data(), lm.data(), lv.data(), lt.data(), soap ? nullptr : nm.data(),
                  soap ? nullptr : nv.data(), soap ? nullptr : nt.data());
    if (soap) {
        int64_t na = 0;
        src.soap_state(nullptr, nullptr, nullptr, nullptr, &na);
        std::vector<double> arena(static_cast<size_t>(na));
        src.soap_state(arena.data(), nm.data(), nv.data(), nt.data(), nullptr);
        dst.set_soap_state(arena.data(), nm.data(), nv.data(), nt.data());
    }
}

bool serial_warmup_forced() {
    static const bool v = [] {
        const char* e = std::getenv("CCB_WARMUP_SERIAL");
        return e && e[0] == '1';
    }();
    return v;
}

}  // namespace

// warmup (encoder.hpp:315-342) with the candidates of each round trained
// CONCURRENTLY ("warm-up candidates are embarrassingly
// parallel"): candidate ci lives in its own trainer (the caller's for ci = 0),
// the round runs as one batched graph (Batch), and every candidate starts from
// the global_iter the sequential loop would give it, so its noise stream —
// and therefore every value — is what the sequential warm-up computes.
// Returns false (state of `tr` reset to a fresh start) when that
// equivalence cannot be guaranteed: a non-finite iteration leaves global_iter
// behind, which shifts the later candidates' noise keys in the sequential
// order; warmup() then runs the sequential loop.
bool warmup_batched(Trainer& tr, const float* image, int h, int w, const cc_decoder_config& dec, int device) {
    const cc_encoder_config& enc = tr.enc();
    const int K = enc.warmup_candidates, it = enc.warmup_iters;
    if (K <= 1 || it <= 0 || serial_warmup_forced()) return false;
    const int64_t g0 = tr.global_iter();
    const int s0 = tr.skipped_steps();
    std::vector<std::unique_ptr<Trainer>> helpers;
    std::vector<Trainer*> all{&tr};
    for (int ci = 1; ci < K; ++ci) {
        helpers.push_back(std::make_unique<Trainer>(image, h, w, enc, dec, device));
        all.push_back(helpers.back().get());
    }
    const size_t nit = static_cast<size_t>(it);
    const std::vector<double> lr(nit, enc.lr_start), tp(nit, enc.temp_start), ns(nit, enc.noise_std_start);
    auto run_round = [&](const std::vector<Trainer*>& ts, const std::vector<int64_t>& start) {
        for (size_t i = 0; i < ts.size(); ++i) ts[i]->set_counters(start[i], 0);
        {
            Batch b(ts);
            b.enqueue_proxy_iterations(it, lr.data(), tp.data(), ns.data());
            b.synchronize();
        }
        bool ok = true;
        for (size_t i = 0; i < ts.size(); ++i) ok = ok && ts[i]->global_iter() == start[i] + it;
        return ok;
    };
    int skipped = 0;
    // round 1: every candidate, fresh (encoder.hpp:317-323)
    std::vector<int64_t> start(static_cast<size_t>(K));
    for (int ci = 0; ci < K; ++ci) {
        all[ci]->fresh_candidate(ci);
        start[size_t(ci)] = g0 + int64_t(ci) * it;
    }
    auto restart = [&] {
        tr.fresh_candidate(0);
        tr.set_counters(g0, s0);
        return false;
    };
    if (!run_round(all, start)) return restart();
    struct C {
        int idx;
        double cost;
    };
    std::vector<C> cands;
    for (int ci = 0; ci < K; ++ci) {
        skipped += all[ci]->skipped_steps();
        cands.push_back({ci, all[ci]->true_cost(nullptr, nullptr)});
    }
    std::stable_sort(cands.begin(), cands.end(), [](const C& a, const C& b) { return a.cost < b.cost; });
    const int keep = std::min<int>(enc.warmup_keep, int(cands.size()));
    cands.resize(size_t(keep));
    // round 2: the kept candidates in sorted order (encoder.hpp:331-336)
    std::vector<Trainer*> kept;
    std::vector<int64_t> start2;
    for (int j = 0; j < keep; ++j) {
        kept.push_back(all[size_t(cands[size_t(j)].idx)]);
        start2.push_back(g0 + int64_t(K + j) * it);
    }
    if (!run_round(kept, start2)) return restart();
    for (int j = 0; j < keep; ++j) {
        skipped += kept[size_t(j)]->skipped_steps();
        cands[size_t(j)].cost = kept[size_t(j)]->true_cost(nullptr, nullptr);
    }
    std::stable_sort(cands.begin(), cands.end(), [](const C& a, const C& b) { return a.cost < b.cost; });
    Trainer* best = all[size_t(cands[0].idx)];
    if (best != &tr) copy_candidate(*best, tr);
    tr.set_counters(g0 + int64_t(K + keep) * it, s0 + skipped);
    tr.set_current_cost(cands[0].cost);
    return true;
}

// warmup (encoder.hpp:315-342): candidates live in device candidate slots.
void warmup(Trainer& tr) {
    const cc_encoder_config& enc = tr.enc();
    struct C {
        int slot;
        double cost;
    };
    std::vector<C> cands;
    for (int ci = 0; ci < enc.warmup_candidates; ++ci) {
        tr.fresh_candidate(ci);
        run_fixed(tr, enc.warmup_iters, enc.lr_start, enc.temp_start, enc.noise_std_start);
        const double c = tr.true_cost(nullptr, nullptr);
        tr.take_candidate(ci, c);
        cands.push_back({ci, c});
    }
    std::stable_sort(cands.begin(), cands.end(), [](const C& a, const C& b) { return a.cost < b.cost; });
    const int keep = std::min<int>(enc.warmup_keep, int(cands.size()));
    if (enc.warmup_candidates <= 1) {
        tr.load_candidate(cands[0].slot);
        return;
    }
    if (keep < int(cands.size())) {
        for (size_t i = size_t(keep); i < cands.size(); ++i) tr.discard_candidate(cands[i].slot);
        cands.resize(size_t(keep));
    }
    for (auto& c : cands) {
        tr.load_candidate(c.slot);
        run_fixed(tr, enc.warmup_iters, enc.lr_start, enc.temp_start, enc.noise_std_start);
        c.cost = tr.true_cost(nullptr, nullptr);
        tr.take_candidate(c.slot, c.cost);
    }
    std::stable_sort(cands.begin(), cands.end(), [](const C& a, const C& b) { return a.cost < b.cost; });
    for (size_t i = 1; i < cands.size(); ++i) tr.discard_candidate(cands[i].slot);
    tr.load_candidate(cands[0].slot);
    tr.set_current_cost(cands[0].cost);
}

// train (encoder.hpp:349-413) on a trainer whose counters were reset.
void train(Trainer& tr, cc_train_stats* out, const float* image, int h, int w, const cc_decoder_config* dec,
           int device) {
    const auto t0 = std::chrono::steady_clock::now();
    const cc_encoder_config& enc = tr.enc();
    const double npix = double(tr.plan().npix);
    Log log(tr.log_path());
    if (!(image && dec && warmup_batched(tr, image, h, w, *dec, device))) warmup(tr);

    const int horizon = std::max(1, enc.main_iters - 1);
    cc_train_stats st{};
    st.true_cost = std::numeric_limits<double>::infinity();
    double lr_scale = 1.0;
    const int kBest = 0;
    tr.snapshot(kBest, tr.true_cost(nullptr, nullptr));

    const int interval = std::max(1, enc.true_cost_interval);
    int it = 0;
    std::vector<double> lr, tp, ns, rec;
    while (it < enc.main_iters) {
        // chunk up to (and including) the next evaluation point
        int last = it;
        while (!((last + 1) % interval == 0 || last == enc.main_iters - 1)) ++last;
        const int n = last - it + 1;
        lr.resize(n);
        tp.resize(n);
        ns.resize(n);
        rec.resize(4 * size_t(n));
        for (int i = 0; i < n; ++i) {
            lr[i] = lr_scale * sched_value(enc.lr_start, enc.lr_end, true, horizon, it + i);
            tp[i] = sched_value(enc.temp_start, enc.temp_end, false, horizon, it + i);
            ns[i] = sched_value(enc.noise_std_start, enc.noise_std_end, false, horizon, it + i);
        }
        tr.proxy_iterations(n, lr.data(), tp.data(), ns.data(), rec.data());
        int bad = -1;
        for (int i = 0; i < n; ++i)
            if (!std::isfinite(rec[4 * size_t(i)])) {
                bad = i;
                break;
            }
        const int ok = bad < 0 ? n : bad;
        for (int i = 0; i < ok; ++i) {
            const double* r = &rec[4 * size_t(i)];
            const bool eval = bad < 0 && i == n - 1;
            if (eval) {
                const double tc = tr.true_cost(nullptr, nullptr);
                if (tc < tr.snapshot_cost(kBest)) tr.snapshot(kBest, tc);
                log.row(int64_t(r[3]), r[0], &tc, r[1], r[2], npix);
            } else {
                log.row(int64_t(r[3]), r[0], nullptr, r[1], r[2], npix);
            }
        }
        if (bad >= 0) {
            // encoder.hpp:365-372 — the later iterations of the chunk were
            // no-ops: k_finalize's sticky halt flag stops every step and
            // counter update after the first non-finite cost of a batch
            if (st.restarts >= 2) break;
            ++st.restarts;
            lr_scale *= 0.5;
            tr.restore(kBest);
            tr.reset_optimizers();
            tr.set_counters(tr.global_iter() + 1, tr.skipped_steps());
            it += bad + 1;
            continue;
        }
        it += n;
    }

    // hardround (encoder.hpp:384-392)
    tr.restore(kBest);
    tr.quantize_all();
    tr.load_pads_from_q();
    for (int i = 0; i < enc.hardround_iters; ++i) {
        const double c = tr.hardround_iteration(enc.hardround_lr, kBest);
        if (!std::isfinite(c)) break;
        log.row(tr.global_iter(), c, &c, tr.last_mse(), tr.last_bits(), npix);
    }
    {
        const double tc = tr.true_cost(nullptr, nullptr);
        if (tc < tr.snapshot_cost(kBest)) tr.snapshot(kBest, tc);
    }
    tr.restore(kBest);
    tr.quantize_all();
    st.iterations = tr.global_iter();
    st.skipped_steps = tr.skipped_steps();
    double psnr = 0.0, bpp = 0.0;
    st.true_cost = tr.true_cost(&psnr, &bpp);
    st.psnr = psnr;
    st.rate_bpp = bpp;
    st.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (out) *out = st;
}

}  // namespace ccb

extern "C" {

const char* cc_last_error(void) { return g_err.c_str(); }
const char* cc_impl_name(void) { return "b200"; }

int cc_decoder_config_preset(const char* name, cc_decoder_config* out) {
    const std::string n = name ? name : "";
    // DecoderConfig::lop/mop/hop/vhop (config.hpp:53-56)
    if (n == "lop") *out = {0, 6, 2, 8, 2, 8, 1, 1, 1};
    else if (n == "mop") *out = {1, 10, 4, 10, 2, 16, 2, 1, 1};
    else if (n == "hop") *out = {2, 14, 6, 20, 2, 48, 2, 1, 1};
    else if (n == "vhop") *out = {3, 20, 6, 26, 2, 64, 2, 1, 1};
    else return fail(CC_ERR_CONFIG, "unknown decoder config: " + n);
    return CC_OK;
}

int cc_encoder_config_default(cc_encoder_config* out) {
    *out = default_enc();
    return CC_OK;
}

int cc_encoder_config_with_total(int total, cc_encoder_config* out) {
    cc_encoder_config cfg = default_enc();
    const int def_total = warmup_total(cfg) + cfg.main_iters + cfg.hardround_iters;
    if (total == def_total) {
        *out = cfg;
        return CC_OK;
    }
    if (total < 20) return fail(CC_ERR_CONFIG, "iteration budget too small");
    const double f = double(total) / 100000.0;
    cfg.warmup_iters = std::max(1, int(std::lround(400.0 * f)));
    cfg.hardround_iters = std::max(1, int(std::lround(500.0 * f)));
    int rest = total - warmup_total(cfg) - cfg.hardround_iters;
    while (rest < 1 && cfg.warmup_iters > 1) {
        --cfg.warmup_iters;
        rest = total - warmup_total(cfg) - cfg.hardround_iters;
    }
    cfg.main_iters = std::max(1, rest);
    *out = cfg;
    return CC_OK;
}

// count_macs_per_pixel (synthesis.hpp:239-277)
double cc_count_macs_per_pixel(const cc_decoder_config* cfg, int H, int W) {
    const int levels = int64_t(H) * int64_t(W) < 1000000 ? 7 : 8;
    const double npix = double(H) * double(W);
    auto cdiv = [](int a, int b) { return (a + b - 1) / b; };
    auto grid_pix = [&](int k) { return double(cdiv(H, 1 << k)) * double(cdiv(W, 1 << k)); };
    const int d = cfg->spatial_ctx + cfg->ifce_dim;
    const int w = cfg->arm_width;
    double arm = double(d) * w + double(w) * w + 2.0 * w;
    if (cfg->use_stabilizer) arm += 2.0 * d;
    double total = 0.0;
    for (int k = 0; k < levels; ++k) total += grid_pix(k) * arm;
    if (cfg->use_hyperlatents)
        for (int k = 4; k < levels; ++k) total += grid_pix(k) * arm;
    if (cfg->ifce_dim > 0) {
        const int hyper = cfg->use_hyperlatents ? levels - 4 : 0;
        for (int k = 0; k < std::min(3, levels); ++k) total += grid_pix(k) * double(hyper + levels - 1 - k) * cfg->ifce_dim;
    }
    for (int k = 1; k < levels; ++k)
        for (int j = k - 1; j >= 0; --j) {
            const double rows_in = cdiv(H, 1 << (j + 1));
            const double rows_out = cdiv(H, 1 << j);
            const double cols_out = cdiv(W, 1 << j);
            total += rows_in * cols_out * 4.0 + rows_out * cols_out * 13.0;
        }
    double syn = double(levels) * cfg->synth_hidden + cfg->synth_hidden * 3.0 + cfg->synth_posts * 81.0;
    if (cfg->use_stabilizer) syn += 3.0 * levels;
    total += npix * syn;
    return total / npix;
}

int cc_make_synthetic_image(int h, int w, uint64_t seed, float* out) {
    if (h < 1 || w < 1) return fail(CC_ERR_CONFIG, "image dimensions must be positive");
    ccs_make_image(h, w, seed, out);
    return CC_OK;
}

int cc_trainer_create(const float* image, int h, int w, const cc_encoder_config* enc,
                      const cc_decoder_config* dec, int device, cc_trainer** out) {
    return guarded([&] {
        auto t = std::make_unique<cc_trainer>();
        t->h = h;
        t->w = w;
        t->enc = *enc;
        t->log_path = enc->log_path ? enc->log_path : "";
        t->enc.log_path = nullptr;
        t->dec = *dec;
        t->device = device;
        if (h < 1 || w < 1) throw ccb::ConfigError("image dimensions must be positive");
        t->image.assign(image, image + size_t(3) * h * w);
        cc_encoder_config e = t->enc;
        e.log_path = t->log_path.c_str();
        t->tr = std::make_unique<Trainer>(image, h, w, e, *dec, device);
        *out = t.release();
        return CC_OK;
    });
}

void cc_trainer_destroy(cc_trainer* t) { delete t; }

int cc_trainer_upload_image(cc_trainer* t, const float* image) {
    return guarded([&] {
        std::memcpy(t->image.data(), image, sizeof(float) * t->image.size());
        t->tr->upload_image(image);
        return CC_OK;
    });
}

int cc_trainer_layout(cc_trainer* t, cc_layout* out) {
    const ccb::Plan& P = t->tr->plan();
    out->height = P.H;
    out->width = P.W;
    out->levels = P.L;
    out->hyper_count = P.hyper;
    out->n_grids = P.n_grids;
    out->n_latents = P.n_latents;
    out->n_tensors = P.n_tensors;
    out->n_params = P.n_params;
    out->pad = P.P;
    return CC_OK;
}

int cc_trainer_grid_info(cc_trainer* t, int gi, cc_grid_info* out) {
    const auto& g = t->tr->grids();
    if (gi < 0 || gi >= int(g.size())) return fail(CC_ERR_CONFIG, "grid index");
    out->level = g[gi].level;
    out->hyper = g[gi].hyper;
    out->rows = g[gi].rows;
    out->cols = g[gi].cols;
    out->offset = g[gi].offset;
    out->ifce_slot = g[gi].ifce_slot;
    return CC_OK;
}

int cc_trainer_param_info(cc_trainer* t, int ti, cc_param_info* out) {
    const auto& ts = t->tr->tensors();
    if (ti < 0 || ti >= int(ts.size())) return fail(CC_ERR_CONFIG, "tensor index");
    std::memset(out->name, 0, sizeof(out->name));
    std::strncpy(out->name, ts[ti].name.c_str(), sizeof(out->name) - 1);
    out->rows = ts[ti].rows;
    out->cols = ts[ti].cols;
    out->size = ts[ti].size;
    out->offset = ts[ti].offset;
    return CC_OK;
}

int cc_trainer_fresh_candidate(cc_trainer* t, int index) {
    return guarded([&] {
        t->tr->fresh_candidate(index);
        return CC_OK;
    });
}

int cc_trainer_set_state(cc_trainer* t, const float* latents, const float* params,
                         const float* lat_m, const float* lat_v, const int64_t* lat_t,
                         const float* nn_m, const float* nn_v, const int64_t* nn_t) {
    return guarded([&] {
        t->tr->set_state(latents, params, lat_m, lat_v, lat_t, nn_m, nn_v, nn_t);
        return CC_OK;
    });
}

int cc_trainer_get_state(cc_trainer* t, float* latents, float* params, float* lat_m,
                         float* lat_v, int64_t* lat_t, float* nn_m, float* nn_v,
                         int64_t* nn_t) {
    return guarded([&] {
        t->tr->get_state(latents, params, lat_m, lat_v, lat_t, nn_m, nn_v, nn_t);
        return CC_OK;
    });
}

int cc_trainer_get_grads(cc_trainer* t, float* lg, float* pg) {
    return guarded([&] {
        t->tr->get_grads(lg, pg);
        return CC_OK;
    });
}

int cc_trainer_get_q(cc_trainer* t, int32_t* q) {
    return guarded([&] {
        t->tr->get_q(q);
        return CC_OK;
    });
}

int cc_trainer_get_counters(cc_trainer* t, int64_t* gi, int* sk) {
    return guarded([&] {
        if (gi) *gi = t->tr->global_iter();
        if (sk) *sk = t->tr->skipped_steps();
        return CC_OK;
    });
}

int cc_trainer_set_counters(cc_trainer* t, int64_t gi, int sk) {
    return guarded([&] {
        t->tr->set_counters(gi, sk);
        return CC_OK;
    });
}

int cc_trainer_proxy_iteration(cc_trainer* t, double lr, double temp, double noise_std,
                               double* cost) {
    return guarded([&] {
        const double c = t->tr->proxy_iteration(lr, temp, noise_std);
        if (cost) *cost = c;
        return CC_OK;
    });
}

int cc_trainer_proxy_iterations(cc_trainer* t, int n, const double* lr, const double* temp,
                                const double* noise_std, double* costs, int* ran) {
    return guarded([&] {
        std::vector<double> rec(4 * size_t(std::max(n, 0)));
        t->tr->proxy_iterations(n, lr, temp, noise_std, rec.data());
        int r = n;
        for (int i = 0; i < n; ++i) {
            if (r == n && !std::isfinite(rec[4 * size_t(i)])) r = i + 1;
            if (costs) costs[i] = i < r ? rec[4 * size_t(i)] : std::nan("");
        }
        if (ran) *ran = r;
        return CC_OK;
    });
}

int cc_trainer_hardround_iteration(cc_trainer* t, double lr, int best_slot, double* cost) {
    return guarded([&] {
        const double c = t->tr->hardround_iteration(lr, best_slot);
        if (cost) *cost = c;
        return CC_OK;
    });
}

int cc_trainer_true_cost(cc_trainer* t, double* cost, double* psnr, double* bpp) {
    return guarded([&] {
        const double c = t->tr->true_cost(psnr, bpp);
        if (cost) *cost = c;
        return CC_OK;
    });
}

int cc_trainer_quantize_all(cc_trainer* t) {
    return guarded([&] {
        t->tr->quantize_all();
        return CC_OK;
    });
}

int cc_trainer_load_pads_from_q(cc_trainer* t) {
    return guarded([&] {
        t->tr->load_pads_from_q();
        return CC_OK;
    });
}

int cc_trainer_last_terms(cc_trainer* t, double* mse, double* bits) {
    if (mse) *mse = t->tr->last_mse();
    if (bits) *bits = t->tr->last_bits();
    return CC_OK;
}

int cc_trainer_snapshot(cc_trainer* t, int slot, double cost) {
    return guarded([&] {
        t->tr->snapshot(slot, cost);
        return CC_OK;
    });
}

int cc_trainer_snapshot_cost(cc_trainer* t, int slot, double* cost) {
    return guarded([&] {
        *cost = t->tr->snapshot_cost(slot);
        return CC_OK;
    });
}

int cc_trainer_restore(cc_trainer* t, int slot) {
    return guarded([&] {
        t->tr->restore(slot);
        return CC_OK;
    });
}

int cc_trainer_reset_optimizers(cc_trainer* t) {
    return guarded([&] {
        t->tr->reset_optimizers();
        return CC_OK;
    });
}

int cc_trainer_take_candidate(cc_trainer* t, int slot, double cost) {
    return guarded([&] {
        t->tr->take_candidate(slot, cost);
        return CC_OK;
    });
}

int cc_trainer_load_candidate(cc_trainer* t, int slot) {
    return guarded([&] {
        t->tr->load_candidate(slot);
        return CC_OK;
    });
}

int cc_trainer_candidate_cost(cc_trainer* t, int slot, double* cost) {
    return guarded([&] {
        *cost = t->tr->candidate_cost(slot);
        return CC_OK;
    });
}

int cc_trainer_set_stream(cc_trainer* t, void* stream) {
    return guarded([&] {
        t->tr->set_stream(static_cast<cudaStream_t>(stream));
        return CC_OK;
    });
}

int cc_trainer_enqueue_proxy_iterations(cc_trainer* t, int n, const double* lr,
                                        const double* temp, const double* noise_std) {
    return guarded([&] {
        t->tr->enqueue_proxy_iterations(n, lr, temp, noise_std);
        return CC_OK;
    });
}

int cc_trainer_reserve_iterations(cc_trainer* t, int n) {
    return guarded([&] {
        t->tr->reserve_iterations(n);
        return CC_OK;
    });
}

int cc_trainer_synchronize(cc_trainer* t) {
    return guarded([&] {
        t->tr->synchronize();
        return CC_OK;
    });
}

int cc_trainer_last_records(cc_trainer* t, int n, double* rec) {
    return guarded([&] {
        t->tr->last_records(n, rec);
        return CC_OK;
    });
}

// ---- diagnostics (include/coolchic_b200_diag.h) ----
const char* ccb_stage_name(int s) {
    static const char* names[] = {"softq_fwd", "arm", "pyramid", "ups_fwd",
                                  "syn_fwd",   "syn_bwd", "ups_bwd", "tail"};
    return (s >= 0 && s < 8) ? names[s] : "?";
}

int ccb_profile_stages(cc_trainer* t, int n, double lr, double temp, double noise, double* ms) {
    return guarded([&] {
        t->tr->profile_stages(n, lr, temp, noise, ms);
        return CC_OK;
    });
}

int ccb_kernels_per_iteration(cc_trainer* t, int* count) {
    return guarded([&] {
        *count = t->tr->kernels_per_iteration();
        return CC_OK;
    });
}

double ccb_arm_flops(cc_trainer* t) {
    const ccb::Plan& P = t->tr->plan();
    double macs = 0.0;
    const double per = double(P.D) * P.Wd + double(P.Wd) * P.Wd + 2.0 * P.Wd +
                       (P.off_astab >= 0 ? 2.0 * P.D : 0.0);
    for (int gi = 0; gi < P.n_grids; ++gi) {
        const double cnt = double(P.g[gi].rows) * P.g[gi].cols;
        macs += cnt * per;
        // IFCE: forward + dF backward in the ARM kernel; its weight gradient
        // is in the ARM kernel too unless k_ifce_dw takes it (Plan::ifce_sep)
        if (P.g[gi].ifce_slot >= 0) macs += cnt * double(P.g[gi].rdim) * P.F * (P.ifce_sep ? 4.0 / 6.0 : 1.0);
    }
    return 6.0 * macs;
}

int ccb_fp32_peak(int device, double* tflops, double* ms) {
    return guarded([&] {
        ccb::fp32_peak(device, tflops, ms);
        return CC_OK;
    });
}

int ccb_eval_math(int fn, int n, const float* a, const float* b, const float* c, float* out) {
    return guarded([&] {
        ccb::eval_math(fn, n, a, b, c, out);
        return CC_OK;
    });
}

int ccb_counter_gauss(uint64_t stream, uint64_t idx0, int n, float* out) {
    return guarded([&] {
        ccb::gauss(stream, idx0, n, out);
        return CC_OK;
    });
}

int ccb_timeline(cc_trainer* t, int n, double lr, double temp, double noise, double* ms) {
    return guarded([&] {
        t->tr->timeline(n, lr, temp, noise, ms);
        return CC_OK;
    });
}

int ccb_soap_state(cc_trainer* t, double* arena, float* m1, float* v2, int64_t* steps, int64_t* n_arena) {
    return guarded([&] {
        t->tr->soap_state(arena, m1, v2, steps, n_arena);
        return CC_OK;
    });
}

int ccb_soap_set_state(cc_trainer* t, const double* arena, const float* m1, const float* v2,
                       const int64_t* steps) {
    return guarded([&] {
        t->tr->set_soap_state(arena, m1, v2, steps);
        return CC_OK;
    });
}

int ccb_host_sync_count(int64_t* n) {
    return guarded([&] {
        *n = ccb::host_sync_count();
        return CC_OK;
    });
}

int cc_trainer_warmup(cc_trainer* t) {
    return guarded([&] {
        if (!ccb::warmup_batched(*t->tr, t->image.data(), t->h, t->w, t->dec, t->device)) ccb::warmup(*t->tr);
        return CC_OK;
    });
}

int cc_trainer_train(cc_trainer* t, cc_train_stats* stats, float* latents, int32_t* q,
                     float* params) {
    return guarded([&] {
        // train() builds a fresh Trainer (encoder.hpp:351): start from scratch
        cc_encoder_config e = t->enc;
        e.log_path = t->log_path.c_str();
        t->tr.reset();
        t->tr = std::make_unique<Trainer>(t->image.data(), t->h, t->w, e, t->dec, t->device);
        ccb::train(*t->tr, stats, t->image.data(), t->h, t->w, &t->dec, t->device);
        if (latents || q || params) {
            std::vector<float> lat(size_t(t->tr->plan().n_latents));
            t->tr->get_state(lat.data(), params, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
            if (latents) std::memcpy(latents, lat.data(), sizeof(float) * lat.size());
            if (q) t->tr->get_q(q);
        }
        return CC_OK;
    });
}

}  // extern "C"

// ---------------------------------------------------------------- row bands
#include "../../include/coolchic_b200_band.h"

extern "C" {

int cc_band_window(int h, int w, int r0, int r1, int halo, int* w0, int* w1) {
    return guarded([&] {
        Trainer::band_window(h, w, r0, r1, halo, w0, w1);
        return CC_OK;
    });
}

int cc_band_trainer_create(const float* image_window, int h, int w, int r0, int r1, int halo,
                           const cc_encoder_config* enc, const cc_decoder_config* dec, int device,
                           cc_trainer** out) {
    return guarded([&] {
        int w0 = 0, w1 = 0;
        Trainer::band_window(h, w, r0, r1, halo, &w0, &w1);
        auto t = std::make_unique<cc_trainer>();
        t->h = w1 - w0;
        t->w = w;
        t->enc = *enc;
        t->log_path = "";
        t->enc.log_path = nullptr;
        t->dec = *dec;
        t->device = device;
        t->image.assign(image_window, image_window + size_t(3) * size_t(w1 - w0) * size_t(w));
        t->tr = std::make_unique<Trainer>(image_window, h, w, r0, r1, halo, t->enc, *dec, device);
        *out = t.release();
        return CC_OK;
    });
}

int cc_band_grid_rows(cc_trainer* t, int gi, int* out4) {
    return guarded([&] {
        if (gi < 0 || gi >= t->tr->plan().n_grids) throw ccb::ConfigError("grid index out of range");
        t->tr->band_grid_rows(gi, out4);
        return CC_OK;
    });
}

int cc_band_rows(cc_trainer* t, int which, int gi, int rb, int re, float* buf, int mode) {
    return guarded([&] {
        t->tr->band_rows(which, gi, rb, re, buf, mode);
        return CC_OK;
    });
}

int cc_band_device_rows(cc_trainer* t, int which, int gi, int rb, int re, void** dptr, int64_t* count) {
    return guarded([&] {
        int64_t n = 0;
        *dptr = t->tr->band_device_rows(which, gi, rb, re, &n);
        if (count) *count = n;
        return CC_OK;
    });
}

int cc_band_device_nn_partial(cc_trainer* t, void** dptr, int64_t* count) {
    return guarded([&] {
        *dptr = t->tr->nn_partial_device();
        if (count) *count = t->tr->plan().n_params;
        return CC_OK;
    });
}

int cc_band_forward_backward(cc_trainer* t, double lr, double temp, double noise_std, double* bits,
                             double* sq_err) {
    return guarded([&] {
        double b = 0.0, s = 0.0;
        t->tr->band_forward_backward(lr, temp, noise_std, &b, &s);
        if (bits) *bits = b;
        if (sq_err) *sq_err = s;
        return CC_OK;
    });
}

int cc_band_nn_partial(cc_trainer* t, double* out) {
    return guarded([&] {
        t->tr->band_nn_partial(out);
        return CC_OK;
    });
}

int cc_band_finish(cc_trainer* t, const double* nn_sums, double bits, double sq_err, double* cost,
                   int* lat_ok_own) {
    return guarded([&] {
        const double c = t->tr->band_finish(nn_sums, bits, sq_err, lat_ok_own);
        if (cost) *cost = c;
        return CC_OK;
    });
}

int cc_band_step(cc_trainer* t, const int* lat_ok) {
    return guarded([&] {
        t->tr->band_step(lat_ok);
        return CC_OK;
    });
}

int cc_band_group_local(cc_trainer* const* bands, int nbands, cc_band_group** out) {
    return guarded([&] {
        if (!bands || nbands < 1 || !out) throw ccb::ConfigError("bad band list");
        std::vector<Trainer*> v;
        for (int b = 0; b < nbands; ++b) {
            if (!bands[b]) throw ccb::ConfigError("null band trainer");
            v.push_back(bands[b]->tr.get());
        }
        auto g = std::make_unique<cc_band_group>();
        g->g = std::make_unique<ccb::BandGroup>(v);
        *out = g.release();
        return CC_OK;
    });
}

int cc_band_nccl_unique_id(void* id128) {
    return guarded([&] {
        if (!id128) throw ccb::ConfigError("null id buffer");
        ccb::BandGroup::nccl_unique_id(id128);
        return CC_OK;
    });
}

int cc_band_group_nccl(cc_trainer* band, const void* id128, int nranks, int rank, const int* edges,
                       cc_band_group** out) {
    return guarded([&] {
        if (!band || !id128 || !edges || !out) throw ccb::ConfigError("null argument");
        auto g = std::make_unique<cc_band_group>();
        g->g = std::make_unique<ccb::BandGroup>(band->tr.get(), id128, nranks, rank, edges);
        *out = g.release();
        return CC_OK;
    });
}

int cc_band_group_reserve(cc_band_group* g, int n) {
    return guarded([&] {
        g->g->reserve(n);
        return CC_OK;
    });
}

int cc_band_group_enqueue_proxy_iterations(cc_band_group* g, int n, const double* lr, const double* temp,
                                           const double* noise_std) {
    return guarded([&] {
        g->g->enqueue_proxy_iterations(n, lr, temp, noise_std);
        return CC_OK;
    });
}

int cc_band_group_synchronize(cc_band_group* g) {
    return guarded([&] {
        g->g->synchronize();
        return CC_OK;
    });
}

int cc_band_group_destroy(cc_band_group* g) {
    return guarded([&] {
        delete g;
        return CC_OK;
    });
}

}  // extern "C"

// ---------------------------------------------------------------- decode passes
#include "../../include/coolchic_b200_codec.h"

extern "C" {

int cc_trainer_set_q(cc_trainer* t, const int32_t* q) {
    return guarded([&] {
        t->tr->set_q(q);
        return CC_OK;
    });
}

int cc_trainer_decode_terms(cc_trainer* t, const float* params, int which, double* rate_bits,
                            double* mse) {
    return guarded([&] {
        if (which < 1 || which > 3) throw ccb::ConfigError("which must be 1 (rate), 2 (mse) or 3");
        t->tr->decode_terms(params, which, rate_bits, mse);
        return CC_OK;
    });
}

int cc_trainer_latent_mu_sigma(cc_trainer* t, const float* params, float* mu, float* sigma) {
    return guarded([&] {
        t->tr->latent_mu_sigma(params, mu, sigma);
        return CC_OK;
    });
}

}  // extern "C"

// ---------------------------------------------------------------- batches (cfg3)
#include "coolchic_b200_batch.h"


extern "C" {

int cc_batch_create(cc_trainer* const* trainers, int n, cc_batch** out) {
    return guarded([&] {
        if (!trainers || n <= 0 || !out) throw ccb::ConfigError("cc_batch_create: no trainers");
        std::vector<ccb::Trainer*> v;
        for (int i = 0; i < n; ++i) {
            if (!trainers[i]) throw ccb::ConfigError("cc_batch_create: null trainer");
            v.push_back(trainers[i]->tr.get());
        }
        auto* b = new cc_batch;
        b->b = std::make_unique<ccb::Batch>(std::move(v));
        *out = b;
        return CC_OK;
    });
}

void cc_batch_destroy(cc_batch* b) { delete b; }

int cc_batch_reserve_iterations(cc_batch* b, int n) {
    return guarded([&] {
        b->b->reserve_iterations(n);
        return CC_OK;
    });
}

int cc_batch_enqueue_proxy_iterations(cc_batch* b, int n, const double* lr, const double* temp,
                                      const double* noise_std) {
    return guarded([&] {
        b->b->enqueue_proxy_iterations(n, lr, temp, noise_std);
        return CC_OK;
    });
}

int cc_batch_synchronize(cc_batch* b) {
    return guarded([&] {
        b->b->synchronize();
        return CC_OK;
    });
}

}  // extern "C"
