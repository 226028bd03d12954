// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (the checker, never shipped).
//
// Compiles the UNMODIFIED reference headers from /root/reference/proj/include
// (read in place, never copied) behind the C ABI of include/coolchic_b200.h,
// so tests and bench.py's reference arm can drive coolcodec::detail::Trainer
// (encoder.hpp:59-306), warmup (encoder.hpp:315-342) and train
// (encoder.hpp:349-413) exactly like the B200 library.  Built by
// oracle/Makefile into oracle/_ref/libccref.so with the reference's own flags
// (-O3 -ffp-contract=fast, proj/CMakeLists.txt:13).  Only tests/, bench.py's
// cpu_baseline/reference leg and __graft_entry__.smoke() may load it.

#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "coolcodec/coolcodec.hpp"
#include "coolchic_b200.h"
#include "coolchic_synth.h"

using namespace coolcodec;

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
    } catch (const ConfigError& e) {
        return fail(CC_ERR_CONFIG, e.what());
    } catch (const FormatError& e) {
        return fail(CC_ERR_FORMAT, e.what());
    } catch (const TrainingError& e) {
        return fail(CC_ERR_TRAINING, e.what());
    } catch (const std::exception& e) {
        return fail(CC_ERR_STATE, e.what());
    }
}

DecoderConfig to_dec(const cc_decoder_config& c) {
    DecoderConfig d;
    d.preset = Preset(uint8_t(c.preset));
    d.spatial_ctx = c.spatial_ctx;
    d.ifce_dim = c.ifce_dim;
    d.arm_width = c.arm_width;
    d.arm_hidden = c.arm_hidden;
    d.synth_hidden = c.synth_hidden;
    d.synth_posts = c.synth_posts;
    d.use_hyperlatents = c.use_hyperlatents != 0;
    d.use_stabilizer = c.use_stabilizer != 0;
    return d;
}

cc_decoder_config from_dec(const DecoderConfig& d) {
    cc_decoder_config c;
    c.preset = int(d.preset);
    c.spatial_ctx = d.spatial_ctx;
    c.ifce_dim = d.ifce_dim;
    c.arm_width = d.arm_width;
    c.arm_hidden = d.arm_hidden;
    c.synth_hidden = d.synth_hidden;
    c.synth_posts = d.synth_posts;
    c.use_hyperlatents = d.use_hyperlatents;
    c.use_stabilizer = d.use_stabilizer;
    return c;
}

EncoderConfig to_enc(const cc_encoder_config& c) {
    EncoderConfig e;
    e.warmup_candidates = c.warmup_candidates;
    e.warmup_keep = c.warmup_keep;
    e.warmup_iters = c.warmup_iters;
    e.main_iters = c.main_iters;
    e.hardround_iters = c.hardround_iters;
    e.lr_start = c.lr_start;
    e.lr_end = c.lr_end;
    e.noise_std_start = c.noise_std_start;
    e.noise_std_end = c.noise_std_end;
    e.temp_start = c.temp_start;
    e.temp_end = c.temp_end;
    e.hardround_lr = c.hardround_lr;
    e.lambda = c.lambda;
    e.seed = c.seed;
    e.use_soap = c.use_soap != 0;
    e.true_cost_interval = c.true_cost_interval;
    e.log_path = c.log_path ? c.log_path : "";
    return e;
}

cc_encoder_config from_enc(const EncoderConfig& e) {
    cc_encoder_config c;
    c.warmup_candidates = e.warmup_candidates;
    c.warmup_keep = e.warmup_keep;
    c.warmup_iters = e.warmup_iters;
    c.main_iters = e.main_iters;
    c.hardround_iters = e.hardround_iters;
    c.lr_start = e.lr_start;
    c.lr_end = e.lr_end;
    c.noise_std_start = e.noise_std_start;
    c.noise_std_end = e.noise_std_end;
    c.temp_start = e.temp_start;
    c.temp_end = e.temp_end;
    c.hardround_lr = e.hardround_lr;
    c.lambda = e.lambda;
    c.seed = e.seed;
    c.use_soap = e.use_soap;
    c.true_cost_interval = e.true_cost_interval;
    c.log_path = nullptr;
    return c;
}

}  // namespace

struct cc_trainer {
    Image img;
    EncoderConfig enc;
    DecoderConfig dec;
    std::string log_path;
    std::unique_ptr<detail::Trainer> tr;
    std::map<int, detail::Snapshot> snaps;
    std::map<int, detail::CandidateState> cands;
    // layout (independent of whether a candidate is loaded)
    LatentSet shape_lat;
    DecoderModel shape_model;
    size_t n_latents = 0, n_params = 0;
    std::vector<double> records;

    detail::CandidateState& cur() {
        if (tr->current().lat.grids.empty())
            throw std::runtime_error("no candidate loaded (call fresh_candidate/load_candidate)");
        return tr->current();
    }
};

extern "C" {

const char* cc_last_error(void) { return g_err.c_str(); }
const char* cc_impl_name(void) { return "reference"; }

int cc_decoder_config_preset(const char* name, cc_decoder_config* out) {
    return guarded([&] {
        *out = from_dec(DecoderConfig::from_name(name ? name : ""));
        return CC_OK;
    });
}

int cc_encoder_config_default(cc_encoder_config* out) {
    *out = from_enc(EncoderConfig{});
    return CC_OK;
}

int cc_encoder_config_with_total(int total, cc_encoder_config* out) {
    return guarded([&] {
        *out = from_enc(EncoderConfig::with_total(total));
        return CC_OK;
    });
}

double cc_count_macs_per_pixel(const cc_decoder_config* cfg, int h, int w) {
    return count_macs_per_pixel(to_dec(*cfg), h, w);
}

int cc_make_synthetic_image(int h, int w, uint64_t seed, float* out) {
    if (h < 1 || w < 1) return fail(CC_ERR_CONFIG, "image dimensions must be positive");
    ccs_make_image(h, w, seed, out);
    return CC_OK;
}

int cc_trainer_create(const float* image, int h, int w, const cc_encoder_config* enc,
                      const cc_decoder_config* dec, int device, cc_trainer** out) {
    (void)device;
    return guarded([&] {
        if (h < 1 || w < 1) throw ConfigError("image dimensions must be positive");
        auto t = std::make_unique<cc_trainer>();
        t->img = Image(h, w);
        std::memcpy(t->img.pix.data(), image, sizeof(float) * t->img.pix.size());
        t->enc = to_enc(*enc);
        t->dec = to_dec(*dec);
        t->tr = std::make_unique<detail::Trainer>(t->img, t->enc, t->dec);
        t->shape_lat = build_latents(h, w, t->dec);
        t->shape_model = make_model(t->dec, h, w);
        t->n_latents = t->shape_lat.total_values();
        t->n_params = param_count(t->shape_model);
        *out = t.release();
        return CC_OK;
    });
}

void cc_trainer_destroy(cc_trainer* tr) { delete tr; }

int cc_trainer_upload_image(cc_trainer* tr, const float* image) {
    std::memcpy(tr->img.pix.data(), image, sizeof(float) * tr->img.pix.size());
    return CC_OK;
}

int cc_trainer_layout(cc_trainer* t, cc_layout* out) {
    out->height = t->img.h;
    out->width = t->img.w;
    out->levels = t->shape_lat.levels;
    out->hyper_count = t->shape_lat.hyper_count;
    out->n_grids = int(t->shape_lat.grids.size());
    out->n_latents = int64_t(t->n_latents);
    int nt = 0;
    for_each_param(t->shape_model, [&](ParamTensor&) { ++nt; });
    out->n_tensors = nt;
    out->n_params = int64_t(t->n_params);
    out->pad = std::max(1, make_context_offsets(t->dec.spatial_ctx).pad);
    return CC_OK;
}

int cc_trainer_grid_info(cc_trainer* t, int gi, cc_grid_info* out) {
    if (gi < 0 || gi >= int(t->shape_lat.grids.size())) return fail(CC_ERR_CONFIG, "grid index");
    int64_t off = 0;
    for (int i = 0; i < gi; ++i) off += int64_t(t->shape_lat.grids[i].count());
    const auto& g = t->shape_lat.grids[gi];
    out->level = g.level;
    out->hyper = g.hyper;
    out->rows = g.rows;
    out->cols = g.cols;
    out->offset = off;
    out->ifce_slot = g.hyper ? -1 : t->shape_model.ifce_slot(g.level);
    return CC_OK;
}

int cc_trainer_param_info(cc_trainer* t, int ti, cc_param_info* out) {
    int i = 0;
    int64_t off = 0;
    bool found = false;
    for_each_param(t->shape_model, [&](ParamTensor& p) {
        if (i == ti) {
            std::memset(out->name, 0, sizeof(out->name));
            std::strncpy(out->name, p.name.c_str(), sizeof(out->name) - 1);
            const MatView mv = MatView::of(p);
            out->rows = mv.rows;
            out->cols = mv.cols;
            out->size = int64_t(p.size());
            out->offset = off;
            found = true;
        }
        off += int64_t(p.size());
        ++i;
    });
    return found ? CC_OK : fail(CC_ERR_CONFIG, "tensor index");
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
        auto& c = t->cur();
        size_t o = 0;
        for (size_t gi = 0; gi < c.lat.grids.size(); ++gi) {
            auto& g = c.lat.grids[gi];
            const size_t n = g.count();
            if (latents) std::copy(latents + o, latents + o + n, g.y.v.begin());
            if (lat_m) std::copy(lat_m + o, lat_m + o + n, c.adam[gi].m.begin());
            if (lat_v) std::copy(lat_v + o, lat_v + o + n, c.adam[gi].v.begin());
            if (lat_t) c.adam[gi].t = lat_t[gi];
            o += n;
        }
        if (c.nn.use_soap && (nn_m || nn_v || nn_t))
            throw ConfigError("optimizer state transfer needs use_soap = false");
        o = 0;
        size_t ti = 0;
        for_each_param(c.model, [&](ParamTensor& p) {
            const size_t n = p.size();
            if (params) std::copy(params + o, params + o + n, p.v.begin());
            if (nn_m) std::copy(nn_m + o, nn_m + o + n, c.nn.adam[ti].m.begin());
            if (nn_v) std::copy(nn_v + o, nn_v + o + n, c.nn.adam[ti].v.begin());
            if (nn_t) c.nn.adam[ti].t = nn_t[ti];
            o += n;
            ++ti;
        });
        return CC_OK;
    });
}

int cc_trainer_get_state(cc_trainer* t, float* latents, float* params, float* lat_m,
                         float* lat_v, int64_t* lat_t, float* nn_m, float* nn_v,
                         int64_t* nn_t) {
    return guarded([&] {
        auto& c = t->cur();
        size_t o = 0;
        for (size_t gi = 0; gi < c.lat.grids.size(); ++gi) {
            auto& g = c.lat.grids[gi];
            if (latents) std::copy(g.y.v.begin(), g.y.v.end(), latents + o);
            if (lat_m) std::copy(c.adam[gi].m.begin(), c.adam[gi].m.end(), lat_m + o);
            if (lat_v) std::copy(c.adam[gi].v.begin(), c.adam[gi].v.end(), lat_v + o);
            if (lat_t) lat_t[gi] = c.adam[gi].t;
            o += g.count();
        }
        if (c.nn.use_soap && (nn_m || nn_v || nn_t))
            throw ConfigError("optimizer state transfer needs use_soap = false");
        o = 0;
        size_t ti = 0;
        for_each_param(c.model, [&](ParamTensor& p) {
            if (params) std::copy(p.v.begin(), p.v.end(), params + o);
            if (nn_m) std::copy(c.nn.adam[ti].m.begin(), c.nn.adam[ti].m.end(), nn_m + o);
            if (nn_v) std::copy(c.nn.adam[ti].v.begin(), c.nn.adam[ti].v.end(), nn_v + o);
            if (nn_t) nn_t[ti] = c.nn.adam[ti].t;
            o += p.size();
            ++ti;
        });
        return CC_OK;
    });
}

int cc_trainer_get_grads(cc_trainer* t, float* latent_grads, float* param_grads) {
    return guarded([&] {
        auto& c = t->cur();
        size_t o = 0;
        for (auto& g : c.lat.grids) {
            if (latent_grads) std::copy(g.y.g.begin(), g.y.g.end(), latent_grads + o);
            o += g.count();
        }
        o = 0;
        for_each_param(c.model, [&](ParamTensor& p) {
            if (param_grads) std::copy(p.g.begin(), p.g.end(), param_grads + o);
            o += p.size();
        });
        return CC_OK;
    });
}

int cc_trainer_get_q(cc_trainer* t, int32_t* q) {
    return guarded([&] {
        auto& c = t->cur();
        size_t o = 0;
        for (auto& g : c.lat.grids) {
            std::copy(g.q.begin(), g.q.end(), q + o);
            o += g.count();
        }
        return CC_OK;
    });
}

int cc_trainer_get_counters(cc_trainer* t, int64_t* gi, int* sk) {
    if (gi) *gi = t->tr->global_iter;
    if (sk) *sk = t->tr->skipped_steps;
    return CC_OK;
}

int cc_trainer_set_counters(cc_trainer* t, int64_t gi, int sk) {
    t->tr->global_iter = gi;
    t->tr->skipped_steps = sk;
    return CC_OK;
}

int cc_trainer_proxy_iteration(cc_trainer* t, double lr, double temp, double noise_std,
                               double* cost) {
    return guarded([&] {
        t->cur();
        const double c = t->tr->proxy_iteration(lr, temp, noise_std);
        if (cost) *cost = c;
        return CC_OK;
    });
}

int cc_trainer_proxy_iterations(cc_trainer* t, int n, const double* lr, const double* temp,
                                const double* noise_std, double* costs, int* ran) {
    return guarded([&] {
        t->cur();
        int i = 0;
        bool dead = false;
        for (; i < n; ++i) {
            if (dead) {
                if (costs) costs[i] = std::nan("");
                continue;
            }
            const double c = t->tr->proxy_iteration(lr[i], temp[i], noise_std[i]);
            if (costs) costs[i] = c;
            if (!std::isfinite(c)) {
                dead = true;
                if (ran) *ran = i + 1;
            }
        }
        if (!dead && ran) *ran = n;
        return CC_OK;
    });
}

int cc_trainer_set_stream(cc_trainer*, void*) { return CC_OK; }

int cc_trainer_enqueue_proxy_iterations(cc_trainer* t, int n, const double* lr,
                                        const double* temp, const double* noise_std) {
    return guarded([&] {
        t->cur();
        t->records.assign(4 * size_t(std::max(n, 0)), 0.0);
        for (int i = 0; i < n; ++i) {
            const double c = t->tr->proxy_iteration(lr[i], temp[i], noise_std[i]);
            double* r = &t->records[4 * size_t(i)];
            r[0] = c;
            r[1] = t->tr->last_mse();
            r[2] = t->tr->last_bits();
            r[3] = double(t->tr->global_iter);
        }
        return CC_OK;
    });
}

int cc_trainer_synchronize(cc_trainer*) { return CC_OK; }
int cc_trainer_reserve_iterations(cc_trainer*, int) { return CC_OK; }

int cc_trainer_last_records(cc_trainer* t, int n, double* rec) {
    if (size_t(n) * 4 > t->records.size()) return fail(CC_ERR_CONFIG, "no such records");
    std::copy(t->records.begin(), t->records.begin() + 4 * size_t(n), rec);
    return CC_OK;
}

int cc_trainer_hardround_iteration(cc_trainer* t, double lr, int best_slot, double* cost) {
    return guarded([&] {
        t->cur();
        detail::Snapshot* best = nullptr;
        if (best_slot >= 0) best = &t->snaps[best_slot];  // default: cost +inf
        const double c = t->tr->hardround_iteration(lr, best);
        if (cost) *cost = c;
        return CC_OK;
    });
}

int cc_trainer_true_cost(cc_trainer* t, double* cost, double* psnr, double* bpp) {
    return guarded([&] {
        t->cur();
        const double c = t->tr->true_cost(psnr, bpp);
        if (cost) *cost = c;
        return CC_OK;
    });
}

int cc_trainer_quantize_all(cc_trainer* t) {
    return guarded([&] {
        quantize_all(t->cur().lat);
        return CC_OK;
    });
}

int cc_trainer_load_pads_from_q(cc_trainer* t) {
    return guarded([&] {
        t->cur();
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
        t->cur();
        t->snaps[slot] = t->tr->snapshot(cost);
        return CC_OK;
    });
}

int cc_trainer_snapshot_cost(cc_trainer* t, int slot, double* cost) {
    auto it = t->snaps.find(slot);
    *cost = it == t->snaps.end() ? std::numeric_limits<double>::infinity() : it->second.cost;
    return CC_OK;
}

int cc_trainer_restore(cc_trainer* t, int slot) {
    return guarded([&] {
        t->cur();
        auto it = t->snaps.find(slot);
        if (it == t->snaps.end() || !it->second.valid) throw std::runtime_error("empty snapshot slot");
        t->tr->restore(it->second);
        return CC_OK;
    });
}

int cc_trainer_reset_optimizers(cc_trainer* t) {
    return guarded([&] {
        t->cur();
        t->tr->reset_optimizers();
        return CC_OK;
    });
}

int cc_trainer_take_candidate(cc_trainer* t, int slot, double cost) {
    return guarded([&] {
        t->cur();
        t->tr->current().cost = cost;
        t->cands[slot] = t->tr->take_candidate();
        return CC_OK;
    });
}

int cc_trainer_load_candidate(cc_trainer* t, int slot) {
    return guarded([&] {
        auto it = t->cands.find(slot);
        if (it == t->cands.end()) throw std::runtime_error("empty candidate slot");
        t->tr->load_candidate(std::move(it->second));
        t->cands.erase(it);
        return CC_OK;
    });
}

int cc_trainer_candidate_cost(cc_trainer* t, int slot, double* cost) {
    auto it = t->cands.find(slot);
    if (it == t->cands.end()) return fail(CC_ERR_STATE, "empty candidate slot");
    *cost = it->second.cost;
    return CC_OK;
}

int cc_trainer_warmup(cc_trainer* t) {
    return guarded([&] {
        t->tr->load_candidate(warmup(*t->tr, t->enc));
        return CC_OK;
    });
}

int cc_trainer_train(cc_trainer* t, cc_train_stats* stats, float* latents, int32_t* q,
                     float* params) {
    return guarded([&] {
        TrainResult r = train(t->img, t->enc, t->dec);
        if (stats) {
            stats->iterations = r.stats.iterations;
            stats->true_cost = r.stats.true_cost;
            stats->psnr = r.stats.psnr;
            stats->rate_bpp = r.stats.rate_bpp;
            stats->restarts = r.stats.restarts;
            stats->skipped_steps = r.stats.skipped_steps;
            stats->seconds = r.stats.seconds;
        }
        size_t o = 0;
        for (auto& g : r.latents.grids) {
            if (latents) std::copy(g.y.v.begin(), g.y.v.end(), latents + o);
            if (q) std::copy(g.q.begin(), g.q.end(), q + o);
            o += g.count();
        }
        o = 0;
        for_each_param(r.model, [&](ParamTensor& p) {
            if (params) std::copy(p.v.begin(), p.v.end(), params + o);
            o += p.size();
        });
        return CC_OK;
    });
}

// ---------------------------------------------------------------------------
// Element-level hooks into the reference's numerics (tests pin the oracle and
// compare the device restatements against these):
//   fn 0 cc_exp(a)  1 cc_log(a)  2 cc_tanh(a)  3 softround_value(a, T=b)
//   4 laplace_bits(a, mu=b, sigma=c)  5 quantize_value(a, amp=255)
//   6 softround derivative (1-tanh^2(d/T)) / (T * 2tanh(1/2T)) at (a, T=b)
// ---------------------------------------------------------------------------
int ccref_eval_math(int fn, int n, const float* a, const float* b, const float* c, float* out) {
    for (int i = 0; i < n; ++i) {
        switch (fn) {
            case 0: out[i] = cc_exp(a[i]); break;
            case 1: out[i] = cc_log(a[i]); break;
            case 2: out[i] = cc_tanh(a[i]); break;
            case 3: out[i] = softround_value(a[i], b[i]); break;
            case 4: out[i] = laplace_bits(a[i], b[i], c[i]); break;
            case 5: out[i] = float(quantize_value(a[i], 255)); break;
            case 6: {
                float x = a[i], y, th, dx = 0.0f, dy = 1.0f;
                softround_forward(&x, &y, &th, 1, b[i]);
                softround_backward(&dy, &th, &dx, 1, b[i]);
                out[i] = dx;
                break;
            }
            default: return fail(CC_ERR_CONFIG, "unknown math function");
        }
    }
    return CC_OK;
}

int ccref_counter_gauss(uint64_t stream, uint64_t idx0, int n, float* out) {
    for (int i = 0; i < n; ++i) out[i] = counter_gauss(stream, idx0 + uint64_t(i));
    return CC_OK;
}

// ---------------------------------------------------------------------------
// Reference-arm helper for bench.py --impl reference: run `threads`
// independent Trainers (one image each, the reference's only multi-core mode,
// tools/coolcodec.cpp:150-171) for `iters` proxy iterations each.  Returns the
// wall seconds of the timed region through *seconds.
// ---------------------------------------------------------------------------
int ccref_parallel_proxy(const float* image, int h, int w, const cc_encoder_config* enc,
                         const cc_decoder_config* dec, int threads, int warm, int iters,
                         double* seconds) {
    return guarded([&] {
        std::vector<std::unique_ptr<cc_trainer>> ts;
        for (int i = 0; i < threads; ++i) {
            cc_trainer* p = nullptr;
            cc_encoder_config e = *enc;
            e.seed = enc->seed + uint64_t(i);
            const int rc = cc_trainer_create(image, h, w, &e, dec, 0, &p);
            if (rc != CC_OK) return rc;
            ts.emplace_back(p);
            ts.back()->tr->fresh_candidate(0);
        }
        auto run = [&](int n) {
            std::vector<std::thread> th;
            for (int i = 0; i < threads; ++i)
                th.emplace_back([&, i] {
                    for (int k = 0; k < n; ++k)
                        ts[i]->tr->proxy_iteration(enc->lr_start, enc->temp_start,
                                                   enc->noise_std_start);
                });
            for (auto& x : th) x.join();
        };
        run(warm);
        const auto t0 = std::chrono::steady_clock::now();
        run(iters);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return CC_OK;
    });
}

}  // extern "C"

// ---------------------------------------------------------------- decode passes
#include "coolchic_b200_codec.h"

extern "C" {

int cc_trainer_set_q(cc_trainer* t, const int32_t* q) {
    return guarded([&] {
        auto& c = t->cur();
        size_t o = 0;
        for (auto& g : c.lat.grids) {
            std::copy(q + o, q + o + g.count(), g.q.begin());
            o += g.count();
        }
        return CC_OK;
    });
}

int cc_trainer_decode_terms(cc_trainer* t, const float* params, int which, double* rate_bits,
                            double* mse) {
    return guarded([&] {
        if (which < 1 || which > 3) throw ConfigError("which must be 1 (rate), 2 (mse) or 3");
        auto& c = t->cur();
        DecoderModel m = c.model;
        if (params) {
            size_t o = 0;
            for_each_param(m, [&](ParamTensor& p) {
                std::copy(params + o, params + o + p.size(), p.v.begin());
                o += p.size();
            });
        }
        if (which & 1) {
            const ContextOffsets ctx = make_context_offsets(t->dec.spatial_ctx);
            *rate_bits = latent_rate_estimate(c.lat, m, ctx);
        }
        if (which & 2) *mse = mse_rgb(reconstruct_image(c.lat, m), t->img);
        return CC_OK;
    });
}

// walk_symbols' (mu, sigma) sequence (bitstream.hpp:106-141), in decode order
int cc_trainer_latent_mu_sigma(cc_trainer* t, const float* params, float* mu, float* sigma) {
    return guarded([&] {
        auto& c = t->cur();
        DecoderModel m = c.model;
        if (params) {
            size_t o = 0;
            for_each_param(m, [&](ParamTensor& p) {
                std::copy(params + o, params + o + p.size(), p.v.begin());
                o += p.size();
            });
        }
        const ContextOffsets ctx = make_context_offsets(t->dec.spatial_ctx);
        const auto arm = make_arm_view(m, false);
        const auto ifces = make_ifce_views(m, false);
        std::vector<float> cbuf(size_t(arm.d), 0.0f);
        size_t i = 0;
        for (size_t gi = 0; gi < c.lat.grids.size(); ++gi) {
            auto& g = c.lat.grids[gi];
            const int slot = g.hyper ? -1 : m.ifce_slot(g.level);
            const int rdim = slot >= 0 ? ifces[size_t(slot)].rdim : 0;
            for (int j = int(ctx.off.size()); j < arm.d; ++j) cbuf[size_t(j)] = 0.0f;
            for (int r = 0; r < g.rows; ++r)
                for (int cc = 0; cc < g.cols; ++cc, ++i) {
                    extract_spatial_context(g.q.data(), g.rows, g.cols, r, cc, ctx, cbuf.data());
                    if (slot >= 0) {
                        float rvec[kMaxFanOut];
                        for (int j = 0; j < rdim; ++j) {
                            const auto& s = c.lat.grids[size_t(j)];
                            const int sh = s.level - g.level;
                            rvec[j] = float(s.q[size_t(r >> sh) * s.cols + (cc >> sh)]);
                        }
                        const auto& fv = ifces[size_t(slot)];
                        for (int j = 0; j < fv.fdim; ++j) {
                            float acc = fv.b[j];
                            const float* wr = fv.w + size_t(j) * rdim;
                            for (int k = 0; k < rdim; ++k) acc += wr[k] * rvec[k];
                            cbuf[ctx.off.size() + size_t(j)] = acc;
                        }
                    }
                    arm_forward_single(arm, cbuf.data(), mu[i], sigma[i]);
                }
        }
        return CC_OK;
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// fp64 TRUTH of one proxy iteration's gradients (test infrastructure).
//
// The reference's compute kernels are templated on the scalar type so its own
// tests can run them in double (entropy_model.hpp:48-50, mathutil.hpp:49-52:
// the double overloads of cc_exp/cc_log/cc_tanh are libm).  This evaluates
// exactly what Trainer::proxy_iteration (encoder.hpp:97-120) computes before
// its optimiser step — soft-quantise (latent.hpp:118-139), rate_pass
// (entropy_model.hpp:180-336), upsample_forward/backward (synthesis.hpp:55-139),
// synthesize_forward/backward (synthesis.hpp:191-233), mse (layers.hpp:643-657)
// — on the trainer's current state, with every kernel instantiated for
// double.  The inputs are the same values the float trainer uses (latents,
// parameters, image, temp / noise_std / rate upstream rounded to float as
// encoder.hpp:98,64 do); only the arithmetic is wider.  Outputs: latent
// gradients (flat layout), parameter gradients (for_each_param order) and
// {cost, mse, bits}.
// ---------------------------------------------------------------------------
extern "C" int ccref_truth_grads(cc_trainer* t, double temp, double noise_std, double* lat_grad,
                                 double* param_grad, double* scalars) {
    return guarded([&] {
        auto& cs = t->cur();
        LatentSet& lat = cs.lat;
        DecoderModel& m = cs.model;
        const int H = t->img.h, W = t->img.w;
        const size_t npix = size_t(H) * W;
        const ContextOffsets ctx = make_context_offsets(t->dec.spatial_ctx);
        const double tf = double(float(temp)), nf = double(float(noise_std));
        const double upstream = double(float(t->enc.lambda / double(npix)));

        // double copies of every parameter tensor (value + grad), by address
        std::map<const ParamTensor*, std::pair<std::vector<double>, std::vector<double>>> P;
        std::vector<const ParamTensor*> order;
        for_each_param(m, [&](ParamTensor& p) {
            auto& e = P[&p];
            e.first.assign(p.v.begin(), p.v.end());
            e.second.assign(p.v.size(), 0.0);
            order.push_back(&p);
        });
        auto V = [&](const ParamTensor& p) -> const double* { return P.at(&p).first.data(); };
        auto G = [&](const ParamTensor& p) -> double* { return P.at(&p).second.data(); };

        ArmView<double> arm;
        arm.d = m.arm.input_dim;
        arm.w = m.arm.width;
        arm.w1 = V(m.arm.l1.w); arm.b1 = V(m.arm.l1.b);
        arm.w2 = V(m.arm.l2.w); arm.b2 = V(m.arm.l2.b);
        arm.w3 = V(m.arm.head.w); arm.b3 = V(m.arm.head.b);
        arm.stab = m.arm.use_stab ? V(m.arm.stab) : nullptr;
        arm.dw1 = G(m.arm.l1.w); arm.db1 = G(m.arm.l1.b);
        arm.dw2 = G(m.arm.l2.w); arm.db2 = G(m.arm.l2.b);
        arm.dw3 = G(m.arm.head.w); arm.db3 = G(m.arm.head.b);
        arm.dstab = m.arm.use_stab ? G(m.arm.stab) : nullptr;
        std::vector<IfceView<double>> ifces;
        for (auto& p : m.ifce) {
            IfceView<double> v;
            v.rdim = p.map.in;
            v.fdim = p.map.out;
            v.w = V(p.map.w); v.b = V(p.map.b);
            v.dw = G(p.map.w); v.db = G(p.map.b);
            ifces.push_back(v);
        }
        std::vector<UpsampleStageView<double>> ups;
        for (auto& s : m.ups) {
            UpsampleStageView<double> v;
            v.k4 = V(s.tconv); v.r3 = V(s.refine);
            v.dk4 = G(s.tconv); v.dr3 = G(s.refine);
            ups.push_back(v);
        }
        SynthesisView<double> sv;
        sv.L = m.syn.in_ch;
        sv.F = m.syn.hidden;
        sv.posts = int(m.syn.post_w.size());
        sv.c1w = V(m.syn.c1.w); sv.c1b = V(m.syn.c1.b);
        sv.c2w = V(m.syn.c2.w); sv.c2b = V(m.syn.c2.b);
        sv.dc1w = G(m.syn.c1.w); sv.dc1b = G(m.syn.c1.b);
        sv.dc2w = G(m.syn.c2.w); sv.dc2b = G(m.syn.c2.b);
        for (int i = 0; i < sv.posts; ++i) {
            sv.pw[i] = V(m.syn.post_w[i]); sv.pb[i] = V(m.syn.post_b[i]);
            sv.dpw[i] = G(m.syn.post_w[i]); sv.dpb[i] = G(m.syn.post_b[i]);
        }
        sv.stab = m.syn.use_stab ? V(m.syn.stab) : nullptr;
        sv.dstab = m.syn.use_stab ? G(m.syn.stab) : nullptr;

        // soft-quantise every grid into its padded double plane
        const int pad = std::max(1, ctx.pad);
        const size_t ng = lat.grids.size();
        std::vector<PaddedGrid<double>> pads(ng);
        std::vector<std::vector<double>> y(ng), th1(ng), th2(ng);
        std::vector<int> slots(ng);
        const uint64_t gi_iter = uint64_t(t->tr->global_iter);
        for (size_t gi = 0; gi < ng; ++gi) {
            auto& g = lat.grids[gi];
            pads[gi].resize(g.rows, g.cols, pad, g.level, g.hyper);
            y[gi].assign(g.y.v.begin(), g.y.v.end());
            th1[gi].assign(g.count(), 0.0);
            th2[gi].assign(g.count(), 0.0);
            slots[gi] = g.hyper ? -1 : m.ifce_slot(g.level);
            const uint64_t stream = hash_combine(hash_combine(t->enc.seed, gi_iter), gi);  // encoder.hpp:213-215
            for (int r = 0; r < g.rows; ++r) {
                const size_t o = size_t(r) * g.cols;
                soft_quantize_forward(y[gi].data() + o, pads[gi].v_at(r, 0), th1[gi].data() + o,
                                      th2[gi].data() + o, size_t(g.cols), tf, nf, stream, o);
            }
        }
        const double bits = rate_pass(pads, ctx, arm, ifces, slots, lat.hyper_count, upstream, true);

        const int L = lat.levels;
        std::vector<PlaneRef<double>> mains(L);
        std::vector<PlaneGrad<double>> dmains(L);
        for (int k = 0; k < L; ++k) {
            auto& p = pads[lat.main_index(k)];
            mains[k] = {p.v_at(0, 0), p.stride(), p.rows, p.cols};
            dmains[k] = {p.g_at(0, 0), p.stride()};
        }
        std::vector<double> z(size_t(L) * npix, 0.0), dz(z.size(), 0.0), xhat(3 * npix, 0.0),
            dx(3 * npix, 0.0), img(t->img.pix.begin(), t->img.pix.end());
        UpsampleCache<double> ucache;
        SynthCache<double> scache;
        upsample_forward(mains, H, W, ups, z.data(), &ucache);
        synthesize_forward(z.data(), L, H, W, sv, xhat.data(), &scache);
        const double mse = mse_forward(xhat.data(), img.data(), xhat.size());
        mse_backward(xhat.data(), img.data(), 1.0, dx.data(), xhat.size());
        synthesize_backward(z.data(), L, H, W, sv, scache, dx.data(), dz.data());
        upsample_backward(mains, H, W, ups, ucache, dz.data(), dmains);

        size_t off = 0;
        for (size_t gi = 0; gi < ng; ++gi) {
            auto& g = lat.grids[gi];
            std::vector<double> dy(g.count(), 0.0);
            for (int r = 0; r < g.rows; ++r) {
                const size_t o = size_t(r) * g.cols;
                soft_quantize_backward(pads[gi].g_at(r, 0), th1[gi].data() + o, th2[gi].data() + o,
                                       dy.data() + o, size_t(g.cols), tf);
            }
            if (lat_grad) std::copy(dy.begin(), dy.end(), lat_grad + off);
            off += g.count();
        }
        size_t po = 0;
        for (const ParamTensor* p : order) {
            const auto& gr = P.at(p).second;
            if (param_grad) std::copy(gr.begin(), gr.end(), param_grad + po);
            po += gr.size();
        }
        if (scalars) {
            scalars[0] = rd_loss(mse, bits / double(npix), t->enc.lambda);
            scalars[1] = mse;
            scalars[2] = bits;
        }
        return CC_OK;
    });
}

// ---------------------------------------------------------------------------
// The reference's SOAP state (optim.hpp:122-141, NnOptimizer::soap) in the
// layout of the product's ccb_soap_state (include/coolchic_b200_diag.h): per
// tensor in for_each_param order L (r x r), R (c x c), QL, QR as doubles; m1,
// v2 flat fp32; step counts.  Test infrastructure for the SOAP lock-step.
// ---------------------------------------------------------------------------
extern "C" int ccb_soap_state(cc_trainer* t, double* arena, float* m1, float* v2, int64_t* steps,
                              int64_t* n_arena) {
    return guarded([&] {
        auto& nn = t->cur().nn;
        if (!nn.use_soap) throw ConfigError("not a SOAP trainer (use_soap = false)");
        size_t a = 0, o = 0;
        for (size_t i = 0; i < nn.soap.size(); ++i) {
            const SoapState& s = nn.soap[i];
            for (const auto* v : {&s.lpre, &s.rpre, &s.ql, &s.qr}) {
                if (arena) std::copy(v->begin(), v->end(), arena + a);
                a += v->size();
            }
            if (m1) std::copy(s.m1.begin(), s.m1.end(), m1 + o);
            if (v2) std::copy(s.v2.begin(), s.v2.end(), v2 + o);
            o += s.m1.size();
            if (steps) steps[i] = s.t;
        }
        if (n_arena) *n_arena = int64_t(a);
        return CC_OK;
    });
}

extern "C" int ccb_soap_set_state(cc_trainer* t, const double* arena, const float* m1, const float* v2,
                                  const int64_t* steps) {
    return guarded([&] {
        auto& nn = t->cur().nn;
        if (!nn.use_soap) throw ConfigError("not a SOAP trainer (use_soap = false)");
        size_t a = 0, o = 0;
        for (size_t i = 0; i < nn.soap.size(); ++i) {
            SoapState& s = nn.soap[i];
            for (auto* v : {&s.lpre, &s.rpre, &s.ql, &s.qr}) {
                if (arena) std::copy(arena + a, arena + a + v->size(), v->begin());
                a += v->size();
            }
            if (m1) std::copy(m1 + o, m1 + o + s.m1.size(), s.m1.begin());
            if (v2) std::copy(v2 + o, v2 + o + s.v2.size(), s.v2.begin());
            o += s.m1.size();
            if (steps) s.t = steps[i];
        }
        return CC_OK;
    });
}
