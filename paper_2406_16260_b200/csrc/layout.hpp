// Clip-engine workspace layout and exchange plan (pure host).
//
// Frame-buffer conventions (all [frames, H*W, C], one frame = H*W*C elements):
//   conv operand  : [hc pre-halo | f_clip own | hc post-halo]          (cf frames)
//   attn operand  : [ha pre-halo | f_clip own | ha post-halo | remote | null] (af frames)
// Halo slots at the video edge stay zero (the reference's zero padding, ops.cpp:94);
// "remote" slots hold the sampled global frames that lie outside this worker's
// synchronised window, in ascending global-index order.
#pragma once

#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/vinf_temporal.h"
#include "host.hpp"

namespace vinf {

constexpr uint32_t kScratchBlocks = 1024;  // >= 2 * SM count partial rows for GN sums

struct Layout {
    explicit Layout(const vinf_engine_desc& desc);

    vinf_engine_desc d;
    uint32_t f_clip = 0, hw = 0, hc = 0, ha = 0, start = 0;
    uint32_t npre_c = 0, npost_c = 0, npre_a = 0, npost_a = 0;
    uint32_t cf = 0, af = 0, n_remote = 0;
    uint32_t null_frame = 0;        // always-zero attn frame: global tokens under ablation
    bool f32 = true;
    uint64_t es = 4, E = 0;
    float scale = 0.f;
    std::vector<uint32_t> gset;
    std::vector<uint32_t> g_frame;  // attn-buffer frame of each global token
    HostTokens tok[4];              // [ablated attention sync * 2 + bias_global]

    uint64_t off_x = 0, off_y = 0, off_tmp = 0, off_u0 = 0, off_u0lo = 0, off_u0f = 0, off_u1 = 0;
    uint64_t off_u2 = 0, off_u2lo = 0, off_u2f = 0, off_qkv = 0, off_ctx = 0, off_ctxlo = 0;
    uint64_t off_sums = 0, off_stats = 0, off_scratch = 0, off_colstats = 0, off_tok[4] = {0, 0, 0, 0};
    // bf16 mode: GroupNorm folded into the projections (engine.cpp stage_gn_apply):
    // W' = W diag(s) [3C][C] bf16, b' = W t [3C] f32, s and t [C] f32
    uint64_t off_wfold = 0, off_gnaff = 0;
    uint64_t scratch_elems = 0, total = 0;

    std::vector<vinf_xfer> xconv, xattn;

    // First global frame of worker w: w*F/N (even split) or floor(w*F/N) (uneven clips)
    uint32_t clip_start(uint32_t w) const {
        return uint32_t(uint64_t(w) * d.frames / d.workers);
    }

   private:
    void build_exchanges();
};

}  // namespace vinf

struct vinf_layout {
    explicit vinf_layout(const vinf_engine_desc& d) : L(d) {}
    vinf::Layout L;
};
