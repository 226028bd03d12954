// tests/cpp/dropin_nncoding.cpp — TEST: the network-parameter quantisation
// search with its decode passes on the GPU (coolcodec::gpu::select_nn_coding,
// include/coolchic_b200.hpp) vs the reference's select_nn_coding
// (nn_coding.hpp:146-224) on the same trained state, and gpu::encode_image vs
// encode_image.  Prints one JSON line; built by `make -C oracle dropin`.
#include <cstdio>

#include "coolcodec/coolcodec.hpp"
#include "coolchic_b200.hpp"
#include "coolchic_synth.h"

int main(int argc, char** argv) {
    using namespace coolcodec;
    const int h = argc > 1 ? std::atoi(argv[1]) : 48;
    const int w = argc > 2 ? std::atoi(argv[2]) : 64;
    const int total = argc > 3 ? std::atoi(argv[3]) : 600;
    Image img(h, w);
    ccs_make_image(h, w, 5, img.pix.data());
    EncoderConfig enc = EncoderConfig::with_total(total);
    enc.lambda = 1e-3;
    enc.seed = 6;
    enc.use_soap = false;
    enc.true_cost_interval = 50;
    const DecoderConfig dcfg = DecoderConfig::lop();
    // one trained state, searched twice
    gpu::Trainer gt(img, enc, dcfg);
    cc_train_stats st{};
    gpu::check(cc_trainer_train(gt.handle(), &st, nullptr, nullptr, nullptr));
    TrainResult tr;
    gt.export_state(tr.latents, tr.model);
    for (auto& g : tr.latents.grids) {
        g.amp = measure_amplitude(g);
        for (auto& q : g.q) q = std::min(std::max(q, -g.amp), g.amp);
    }
    gt.set_q(tr.latents);
    const ContextOffsets ctx = make_context_offsets(dcfg.spatial_ctx);
    DecoderModel m_ref = tr.model, m_gpu = tr.model;
    const NnCodingResult r = select_nn_coding(img, tr.latents, m_ref, enc.lambda, ctx);
    const NnCodingResult g = gpu::select_nn_coding(gt, tr.latents, m_gpu, enc.lambda);
    int same = 1;
    for (int s = 0; s < kSubmoduleCount; ++s)
        for (int p = 0; p < 2; ++p)
            same &= r.spec.parts[s][p].delta_idx == g.spec.parts[s][p].delta_idx &&
                    r.spec.parts[s][p].kappa == g.spec.parts[s][p].kappa;
    const int same_payload = r.payload == g.payload;
    // latent entropy coding with the device's (mu, sigma): byte-identical
    // payload, and the reference decoder recovers every q from it
    const std::vector<uint8_t> lat_ref = encode_latents(tr.latents, m_ref, ctx);
    const std::vector<uint8_t> lat_gpu = gpu::encode_latents(gt, tr.latents, m_gpu);
    LatentSet back = tr.latents;
    for (auto& gq : back.grids) std::fill(gq.q.begin(), gq.q.end(), 0);
    decode_latents(back, m_ref, ctx, lat_gpu.data(), lat_gpu.size());
    int decodes = 1;
    for (size_t k = 0; k < back.grids.size(); ++k) decodes &= back.grids[k].q == tr.latents.grids[k].q;
    const int same_latent_payload = lat_ref == lat_gpu;
    const EncodeResult e = gpu::encode_image(img, enc, dcfg);
    const int encode_decodes = [&] {
        const DecodeResult d = decode_image(e.bytes);
        return int(d.img.h == img.h && d.img.w == img.w && psnr_rgb(img, d.img) == e.stats.psnr);
    }();
    std::printf(
        "{\"same_spec\": %d, \"same_payload\": %d, \"ref_cost\": %.12g, \"gpu_cost\": %.12g, "
        "\"ref_rate\": %.12g, \"gpu_rate\": %.12g, \"ref_mse\": %.12g, \"gpu_mse\": %.12g, "
        "\"encode_bytes\": %zu, \"encode_psnr\": %.6g, \"encode_bpp\": %.6g, "
        "\"same_latent_payload\": %d, \"latent_decodes\": %d, \"latent_bytes\": %zu, "
        "\"encode_decodes\": %d}\n",
        same, same_payload, r.cost, g.cost, r.rate_bits, g.rate_bits, r.mse, g.mse, e.bytes.size(),
        e.stats.psnr, e.stats.bpp, same_latent_payload, decodes, lat_gpu.size(), encode_decodes);
    return 0;
}
