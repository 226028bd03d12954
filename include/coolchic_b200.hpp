// coolchic_b200.hpp — drop-in C++ surface of the B200 encode loop for code
// that already uses the reference library (proj/include/coolcodec).
//
// Include AFTER the reference headers.  Everything here is a thin, header-only
// shim over the C ABI (coolchic_b200.h); no reference source is compiled into
// libcoolchic_b200.so.  Names and signatures mirror
//   coolcodec::detail::Trainer   (encoder.hpp:59-306)
//   coolcodec::warmup / train    (encoder.hpp:315-413)
// so switching an encoder to the GPU is a namespace change:
//   coolcodec::TrainResult r = coolcodec::gpu::train(img, enc, dcfg);
// Errors come back as the reference's exception types (tensor.hpp:11-25).
#pragma once

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "coolchic_b200.h"

namespace coolcodec {
namespace gpu {

inline void check(int rc) {
    if (rc == CC_OK) return;
    const std::string msg = cc_last_error();
    switch (rc) {
        case CC_ERR_CONFIG: throw ConfigError(msg);
        case CC_ERR_FORMAT: throw FormatError(msg);
        case CC_ERR_TRAINING: throw TrainingError(msg);
        default: throw CodecError(msg);
    }
}

inline cc_decoder_config to_c(const DecoderConfig& d) {
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

inline cc_encoder_config to_c(const EncoderConfig& e) {
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
    c.log_path = e.log_path.c_str();
    return c;
}

// detail::Trainer on the GPU.  Latents/model live on the device; current()
// materialises a CandidateState-shaped host copy on demand.
class Trainer {
public:
    Trainer(const Image& img, const EncoderConfig& enc, const DecoderConfig& dcfg,
            int device = 0)
        : enc_(enc), dcfg_(dcfg) {
        cc_encoder_config ec = to_c(enc_);
        cc_decoder_config dc = to_c(dcfg_);
        check(cc_trainer_create(img.pix.data(), img.h, img.w, &ec, &dc, device, &t_));
        check(cc_trainer_layout(t_, &layout_));
    }
    ~Trainer() { cc_trainer_destroy(t_); }
    Trainer(const Trainer&) = delete;
    Trainer& operator=(const Trainer&) = delete;

    void fresh_candidate(int index) { check(cc_trainer_fresh_candidate(t_, index)); }
    double proxy_iteration(double lr, double temp, double noise_std) {
        double c = 0.0;
        check(cc_trainer_proxy_iteration(t_, lr, temp, noise_std, &c));
        return c;
    }
    // best_slot < 0: no snapshot (the reference's best == nullptr)
    double hardround_iteration(double lr, int best_slot = -1) {
        double c = 0.0;
        check(cc_trainer_hardround_iteration(t_, lr, best_slot, &c));
        return c;
    }
    double true_cost(double* psnr = nullptr, double* bpp = nullptr) {
        double c = 0.0;
        check(cc_trainer_true_cost(t_, &c, psnr, bpp));
        return c;
    }
    void load_pads_from_q() { check(cc_trainer_load_pads_from_q(t_)); }
    void quantize_all() { check(cc_trainer_quantize_all(t_)); }
    void snapshot(int slot, double cost) { check(cc_trainer_snapshot(t_, slot, cost)); }
    void restore(int slot) { check(cc_trainer_restore(t_, slot)); }
    void reset_optimizers() { check(cc_trainer_reset_optimizers(t_)); }
    double last_mse() const {
        double m = 0, b = 0;
        cc_trainer_last_terms(t_, &m, &b);
        return m;
    }
    double last_bits() const {
        double m = 0, b = 0;
        cc_trainer_last_terms(t_, &m, &b);
        return b;
    }
    int64_t global_iter() const {
        int64_t g = 0;
        int s = 0;
        check(cc_trainer_get_counters(t_, &g, &s));
        return g;
    }
    int skipped_steps() const {
        int64_t g = 0;
        int s = 0;
        check(cc_trainer_get_counters(t_, &g, &s));
        return s;
    }

    // Copy the device state into the reference's containers (LatentSet with y
    // and q per grid, DecoderModel in for_each_param order).
    void export_state(LatentSet& lat, DecoderModel& model) {
        lat = build_latents(layout_.height, layout_.width, dcfg_);
        model = make_model(dcfg_, layout_.height, layout_.width);
        std::vector<float> y(size_t(layout_.n_latents)), p(size_t(layout_.n_params));
        std::vector<int32_t> q(size_t(layout_.n_latents));
        check(cc_trainer_get_state(t_, y.data(), p.data(), nullptr, nullptr, nullptr, nullptr,
                                   nullptr, nullptr));
        check(cc_trainer_get_q(t_, q.data()));
        size_t o = 0;
        for (auto& g : lat.grids) {
            std::copy(y.begin() + o, y.begin() + o + g.count(), g.y.v.begin());
            std::copy(q.begin() + o, q.begin() + o + g.count(), g.q.begin());
            o += g.count();
        }
        o = 0;
        for_each_param(model, [&](ParamTensor& t) {
            std::copy(p.begin() + o, p.begin() + o + t.size(), t.v.begin());
            o += t.size();
        });
    }

    cc_trainer* handle() { return t_; }

private:
    EncoderConfig enc_;
    DecoderConfig dcfg_;
    cc_trainer* t_ = nullptr;
    cc_layout layout_{};
};

// train(img, enc, dcfg) (encoder.hpp:349-413): the whole schedule runs inside
// the library (warm-up candidates, main stage in graph replays between
// true-cost checks, restarts, hardround).
inline TrainResult train(const Image& img, const EncoderConfig& enc, const DecoderConfig& dcfg,
                         int device = 0) {
    Trainer tr(img, enc, dcfg, device);
    cc_train_stats st{};
    check(cc_trainer_train(tr.handle(), &st, nullptr, nullptr, nullptr));
    TrainResult r;
    tr.export_state(r.latents, r.model);
    r.stats.iterations = st.iterations;
    r.stats.true_cost = st.true_cost;
    r.stats.psnr = st.psnr;
    r.stats.rate_bpp = st.rate_bpp;
    r.stats.restarts = st.restarts;
    r.stats.skipped_steps = st.skipped_steps;
    r.stats.seconds = st.seconds;
    return r;
}

}  // namespace gpu
}  // namespace coolcodec
