// coolchic_b200.hpp — drop-in C++ surface of the B200 encode loop for code
// that already uses the reference library (proj/include/coolcodec).
//
// Include AFTER the reference headers.  Everything here is a thin, header-only
// shim over the C ABI (coolchic_b200.h); no reference source is compiled into
// libcoolchic_b200.so.  Names and signatures mirror
//   coolcodec::detail::Trainer   (encoder.hpp:59-306)
//   coolcodec::warmup / train    (encoder.hpp:315-413)
//   coolcodec::select_nn_coding  (nn_coding.hpp:146-224), its decode passes on the GPU
//   coolcodec::encode_image      (bitstream.hpp:187-228)
// so switching an encoder to the GPU is a namespace change:
//   coolcodec::TrainResult r = coolcodec::gpu::train(img, enc, dcfg);
// Errors come back as the reference's exception types (tensor.hpp:11-25).
#pragma once

#include <algorithm>
#include <chrono>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "coolchic_b200.h"
#include "coolchic_b200_codec.h"

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

    // forward-only decode passes (decode_core.hpp:38-63) on the device
    void set_q(const LatentSet& lat) {
        std::vector<int32_t> q;
        q.reserve(size_t(layout_.n_latents));
        for (const auto& g : lat.grids) q.insert(q.end(), g.q.begin(), g.q.end());
        check(cc_trainer_set_q(t_, q.data()));
    }
    // which: 1 = latent_rate_estimate, 2 = mse_rgb(reconstruct_image), 3 = both
    void decode_terms(DecoderModel& m, int which, double* rate_bits, double* mse) {
        std::vector<float> p;
        p.reserve(size_t(layout_.n_params));
        for_each_param(m, [&](ParamTensor& t) { p.insert(p.end(), t.v.begin(), t.v.end()); });
        check(cc_trainer_decode_terms(t_, p.data(), which, rate_bits, mse));
    }

    // encode_latents' (mu, sigma) of every quantised latent (decode order),
    // with m's parameters substituted
    void latent_mu_sigma(DecoderModel& m, std::vector<float>& mu, std::vector<float>& sigma) {
        std::vector<float> p;
        p.reserve(size_t(layout_.n_params));
        for_each_param(m, [&](ParamTensor& t) { p.insert(p.end(), t.v.begin(), t.v.end()); });
        mu.resize(size_t(layout_.n_latents));
        sigma.resize(size_t(layout_.n_latents));
        check(cc_trainer_latent_mu_sigma(t_, p.data(), mu.data(), sigma.data()));
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

// select_nn_coding (nn_coding.hpp:146-224) with every candidate evaluation —
// a latent-rate estimate for ARM / IFCE candidates, a reconstruction MSE for
// synthesis / upsampling candidates — done by the trainer's device decode
// passes on its quantised latents (set with Trainer::set_q).  The search
// order, tie rule (strict improvement, coarse-to-fine) and the bit accounting
// are the reference's, through its own helpers.
inline NnCodingResult select_nn_coding(Trainer& tr, const LatentSet& lat, DecoderModel& m,
                                       double lambda) {
    const double npix = double(lat.image_h) * double(lat.image_w);
    NnCodingResult res;
    double cur_rate = 0.0, cur_mse = 0.0, nn_bits = 0.0;
    tr.decode_terms(m, 3, &cur_rate, &cur_mse);
    for (int s = 0; s < kSubmoduleCount; ++s) {
        const Submodule sub = Submodule(s);
        const int which = (sub == Submodule::Arm || sub == Submodule::Ifce) ? 1 : 2;
        auto sp = submodule_params(m, sub);
        std::vector<std::vector<float>> keep_w, keep_b;
        for (auto* t : sp.weights) keep_w.push_back(t->v);
        for (auto* t : sp.biases) keep_b.push_back(t->v);
        auto put_back = [&]() {
            for (size_t i = 0; i < sp.weights.size(); ++i) sp.weights[i]->v = keep_w[i];
            for (size_t i = 0; i < sp.biases.size(); ++i) sp.biases[i]->v = keep_b[i];
        };
        double best = std::numeric_limits<double>::infinity();
        NnPartSpec bw, bb;
        double b_rate = cur_rate, b_mse = cur_mse, b_bits = 0.0;
        for (int iw = 0; iw < kNnDeltaCount; ++iw) {
            const double dw = nn_delta_from_index(iw);
            const auto qw = nn_detail::quantize_part(sp.weights, dw);
            size_t wbits = 0;
            const int kw = nn_detail::best_kappa(qw, &wbits);
            for (int ib = 0; ib < kNnDeltaCount; ++ib) {
                const double db = nn_delta_from_index(ib);
                const auto qb = nn_detail::quantize_part(sp.biases, db);
                size_t bbits = 0;
                const int kb = nn_detail::best_kappa(qb, &bbits);
                nn_detail::apply_dequant(sp.weights, qw, dw);
                nn_detail::apply_dequant(sp.biases, qb, db);
                double rate = cur_rate, mse = cur_mse;
                tr.decode_terms(m, which, &rate, &mse);
                const double bits = double(wbits + bbits) + 2.0 * double(nn_detail::kPartHeaderBits);
                const double cost = mse + lambda * (rate + nn_bits + bits) / npix;
                if (cost < best) {
                    best = cost;
                    bw = {iw, kw};
                    bb = {ib, kb};
                    b_rate = rate;
                    b_mse = mse;
                    b_bits = bits;
                }
                put_back();
            }
        }
        nn_detail::apply_dequant(sp.weights,
                                 nn_detail::quantize_part(sp.weights, nn_delta_from_index(bw.delta_idx)),
                                 nn_delta_from_index(bw.delta_idx));
        nn_detail::apply_dequant(sp.biases,
                                 nn_detail::quantize_part(sp.biases, nn_delta_from_index(bb.delta_idx)),
                                 nn_delta_from_index(bb.delta_idx));
        res.spec.parts[size_t(s)][0] = bw;
        res.spec.parts[size_t(s)][1] = bb;
        nn_bits += b_bits;
        cur_rate = b_rate;
        cur_mse = b_mse;
    }
    res.payload = write_nn_payload(m, res.spec);
    res.rate_bits = cur_rate;
    res.mse = cur_mse;
    res.cost = cur_mse + lambda * (cur_rate + 8.0 * double(res.payload.size())) / npix;
    return res;
}

// encode_latents (bitstream.hpp:145-155) with the per-latent Laplace
// parameters computed on the device for all latents at once (the trainer's q,
// set with Trainer::set_q, and m's parameters); the CDF quantisation
// (quantize_cdf, range_coder.hpp:119-161) and the range coder stay the
// reference's, in walk_symbols' order, so the payload is byte-identical.
inline std::vector<uint8_t> encode_latents(Trainer& tr, LatentSet& set, DecoderModel& m) {
    std::vector<float> mu, sigma;
    tr.latent_mu_sigma(m, mu, sigma);
    RangeEncoder enc;
    std::vector<uint32_t> cum;
    size_t i = 0;
    for (auto& g : set.grids)
        for (size_t k = 0; k < g.q.size(); ++k, ++i) {
            quantize_cdf(mu[i], sigma[i], g.amp, cum);
            const int sym = int(g.q[k]) + g.amp;
            enc.encode(cum[size_t(sym)], cum[size_t(sym) + 1] - cum[size_t(sym)]);
        }
    return enc.finish();
}

// encode_image (bitstream.hpp:187-228): training, the NN-coding search and the
// latents' (mu, sigma) on the GPU; the CDF quantisation, the range coder and
// the bitstream assembly are the reference's.
inline EncodeResult encode_image(const Image& img, const EncoderConfig& enc,
                                 const DecoderConfig& dcfg, int device = 0) {
    const auto t0 = std::chrono::steady_clock::now();
    if (img.h > 0xFFFF || img.w > 0xFFFF) throw ConfigError("image too large for header");
    Trainer gt(img, enc, dcfg, device);
    cc_train_stats st{};
    check(cc_trainer_train(gt.handle(), &st, nullptr, nullptr, nullptr));
    TrainResult tr;
    gt.export_state(tr.latents, tr.model);
    const ContextOffsets ctx = make_context_offsets(dcfg.spatial_ctx);
    for (auto& g : tr.latents.grids) {
        g.amp = measure_amplitude(g);
        for (auto& q : g.q) q = std::min(std::max(q, -g.amp), g.amp);
    }
    gt.set_q(tr.latents);
    NnCodingResult nn = select_nn_coding(gt, tr.latents, tr.model, enc.lambda);
    const std::vector<uint8_t> latent_payload = encode_latents(gt, tr.latents, tr.model);
    BitstreamHeader h;
    h.height = uint16_t(img.h);
    h.width = uint16_t(img.w);
    h.config_id = uint8_t(dcfg.preset);
    for (const auto& g : tr.latents.grids) h.amps.push_back(uint8_t(g.amp));
    h.nn_bytes = uint32_t(nn.payload.size());
    h.latent_bytes = uint32_t(latent_payload.size());
    EncodeResult res;
    res.bytes = write_header(h);
    res.bytes.insert(res.bytes.end(), nn.payload.begin(), nn.payload.end());
    res.bytes.insert(res.bytes.end(), latent_payload.begin(), latent_payload.end());
    res.recon = reconstruct_image(tr.latents, tr.model);
    res.stats.file_bytes = res.bytes.size();
    res.stats.nn_bytes = nn.payload.size();
    res.stats.latent_bytes = latent_payload.size();
    res.stats.bpp = 8.0 * double(res.bytes.size()) / (double(img.h) * double(img.w));
    res.stats.psnr = psnr_rgb(img, res.recon);
    res.stats.latent_rate_estimate_bits = total_rate_bits(tr.latents, tr.model, ctx);
    res.stats.iterations = st.iterations;
    res.stats.restarts = st.restarts;
    res.stats.macs_per_pixel = count_macs_per_pixel(dcfg, img.h, img.w);
    res.stats.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return res;
}

}  // namespace gpu
}  // namespace coolcodec
