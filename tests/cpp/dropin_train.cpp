// tests/cpp/dropin_train.cpp — TEST: the C++ drop-in (include/coolchic_b200.hpp)
// compiled against the reference headers, exactly as an encoder using
// coolcodec would include it.  Runs coolcodec::train (CPU reference) and
// coolcodec::gpu::train (B200) on the same image and prints both results as
// one JSON line.  Built by `make -C oracle dropin` (needs /root/reference once);
// the binary travels to the GPU box, where tests/test_dropin.py runs it.
#include <cstdio>

#include "coolcodec/coolcodec.hpp"
#include "coolchic_b200.hpp"
#include "coolchic_synth.h"

int main(int argc, char** argv) {
    using namespace coolcodec;
    const int h = argc > 1 ? std::atoi(argv[1]) : 40;
    const int w = argc > 2 ? std::atoi(argv[2]) : 48;
    const int total = argc > 3 ? std::atoi(argv[3]) : 600;
    Image img(h, w);
    ccs_make_image(h, w, 3, img.pix.data());
    EncoderConfig enc = EncoderConfig::with_total(total);
    enc.lambda = 1e-3;
    enc.seed = 4;
    enc.use_soap = false;
    enc.true_cost_interval = 50;
    const DecoderConfig dcfg = DecoderConfig::lop();
    const TrainResult ref = train(img, enc, dcfg);
    const TrainResult gpu = gpu::train(img, enc, dcfg);
    size_t nq = 0, qdiff = 0;
    for (size_t gi = 0; gi < ref.latents.grids.size(); ++gi)
        for (size_t i = 0; i < ref.latents.grids[gi].q.size(); ++i) {
            ++nq;
            qdiff += ref.latents.grids[gi].q[i] != gpu.latents.grids[gi].q[i];
        }
    std::printf(
        "{\"ref_cost\": %.9g, \"gpu_cost\": %.9g, \"ref_iters\": %lld, \"gpu_iters\": %lld, "
        "\"ref_psnr\": %.6g, \"gpu_psnr\": %.6g, \"ref_bpp\": %.6g, \"gpu_bpp\": %.6g, "
        "\"q_total\": %zu, \"q_differ\": %zu}\n",
        ref.stats.true_cost, gpu.stats.true_cost, (long long)ref.stats.iterations,
        (long long)gpu.stats.iterations, ref.stats.psnr, gpu.stats.psnr, ref.stats.rate_bpp,
        gpu.stats.rate_bpp, nq, qdiff);
    return 0;
}
