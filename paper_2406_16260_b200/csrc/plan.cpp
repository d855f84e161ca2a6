// Pure-host, integer-exact parts of the path: token sets (ops.cpp:177-198), the clip
// plan (clip_parallel.cpp:54-91), traffic closed forms (clip_parallel.cpp:343-387), and
// the clip engine's workspace layout + exchange plan. No CUDA calls in this file, so
// layouts and exchange plans can be built and tested on CPU-only hosts.
#include <algorithm>
#include <cstring>

#include "host.hpp"
#include "layout.hpp"

namespace vinf {

std::vector<uint32_t> build_local_window(uint32_t a, uint32_t frames, uint32_t n_local) {
    if (a >= frames) range_error("query frame outside video");
    const uint32_t half = n_local / 2;
    const uint32_t lo = a > half ? a - half : 0;
    const uint32_t hi = (a + half < frames) ? a + half : frames - 1;
    std::vector<uint32_t> w;
    w.reserve(hi - lo + 1);
    for (uint32_t i = lo; i <= hi; ++i) w.push_back(i);
    return w;
}

std::vector<uint32_t> build_global_index_set(uint32_t frames, uint32_t n_global) {
    if (n_global > frames)
        config_error("global set size exceeds frame count: " + std::to_string(n_global) + " > " +
                     std::to_string(frames));
    std::vector<uint32_t> idx(n_global);
    for (uint32_t j = 0; j < n_global; ++j) idx[j] = uint32_t((uint64_t(j) * frames) / n_global);
    return idx;
}

uint32_t make_plan(uint32_t frames, uint32_t workers) {
    if (workers == 0) config_error("worker count must be >= 1");
    if (frames == 0 || frames % workers != 0)
        config_error("workers must divide frames evenly: frames=" + std::to_string(frames) +
                     " workers=" + std::to_string(workers));
    return frames / workers;
}

std::vector<uint32_t> global_members_in_range(uint32_t frames, uint32_t n_global, uint32_t start,
                                              uint32_t len) {
    std::vector<uint32_t> local;
    for (uint32_t g : build_global_index_set(frames, n_global))
        if (g >= start && g < start + len) local.push_back(g - start);
    return local;
}

void predict_sync_traffic(uint32_t frames, uint32_t workers, uint32_t halo, uint32_t gframes,
                          uint32_t worker, uint64_t frame_bytes, uint64_t out[3]) {
    const uint32_t f_clip = make_plan(frames, workers);
    out[0] = out[1] = out[2] = 0;
    if (workers == 1) return;
    if (gframes > 0) {
        // ring all-gather: worker i forwards every block except the one from i+1
        uint64_t total = 0, next = 0, mine = 0;
        for (uint32_t w = 0; w < workers; ++w) {
            const uint64_t b =
                global_members_in_range(frames, gframes, w * f_clip, f_clip).size() * frame_bytes;
            total += b;
            if (w == (worker + 1) % workers) next = b;
            if (w == worker) mine = b;
        }
        out[0] += total - next;
        out[1] += mine;
        out[2] += workers - 1;
    }
    if (halo > 0) {
        const uint64_t hb = uint64_t(halo) * frame_bytes;
        if (worker + 1 < workers) { out[0] += hb; out[1] += hb; out[2] += 1; }
        if (worker > 0) { out[0] += hb; out[1] += hb; out[2] += 1; }
    }
}

void predict_groupnorm_traffic(uint32_t frames, uint32_t workers, uint32_t groups,
                               uint64_t out[3]) {
    make_plan(frames, workers);
    out[0] = out[1] = out[2] = 0;
    if (workers == 1) return;
    const uint64_t block = uint64_t(groups) * sizeof(double);
    out[0] = 2 * block * (workers - 1);
    out[1] = 2 * block;
    out[2] = 2 * uint64_t(workers - 1);
}

// ---------------------------------------------------------------------------
// Token tables

void HostTokens::finalize(bool gather4) {
    kv_ok = true;
    wflag = gflag = -1;
    for (uint32_t qb = 0; qb < nqb; ++qb) {
        std::vector<uint16_t> uniq;
        const uint32_t a1 = std::min<uint32_t>(nq, (qb + 1) * kQBlock);
        for (uint32_t a = qb * kQBlock; a < a1; ++a)
            for (uint32_t i = 0; i < count[a]; ++i) uniq.push_back(rows[size_t(a) * kMaxTokens + i]);
        std::sort(uniq.begin(), uniq.end());
        uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
        if (uniq.size() > size_t(kKvMax)) {
            kv_ok = false;
            kv_count[qb] = 0;
            continue;
        }
        kv_count[qb] = uint16_t(uniq.size());
        for (size_t r = 0; r < uniq.size(); ++r) kv_frames[size_t(qb) * kKvMax + r] = uniq[r];
        for (uint32_t a = qb * kQBlock; a < a1; ++a)
            for (uint32_t i = 0; i < count[a]; ++i) {
                const uint16_t row = rows[size_t(a) * kMaxTokens + i];
                col[size_t(a) * kMaxTokens + i] =
                    uint8_t(std::lower_bound(uniq.begin(), uniq.end(), row) - uniq.begin());
            }
        // per-column form: the window is a contiguous frame range, hence a contiguous
        // column range of the sorted list; the global tokens are counted per column
        for (uint32_t a = qb * kQBlock; a < a1; ++a) {
            const uint8_t* c = &col[size_t(a) * kMaxTokens];
            const uint8_t* f = &biased[size_t(a) * kMaxTokens];
            const uint32_t nw = nwin[a], n = count[a];
            if (nw == 0) config_error("every query needs at least one window token");
            wlo[a] = c[0];
            whi[a] = c[nw - 1];
            if (uint32_t(whi[a] - wlo[a] + 1) != nw) config_error("window tokens must be contiguous frames");
            for (uint32_t i = 0; i < n; ++i) {
                const bool is_w = i < nw;
                int& flag = is_w ? wflag : gflag;
                if (flag == -1) flag = f[i];
                if (flag != f[i]) config_error("bias flags must be uniform per token kind");
                if (is_w && i > 0 && c[i] != c[i - 1] + 1) config_error("window tokens must be ascending");
            }
            if (a == qb * kQBlock) {
                for (uint32_t i = nw; i < n; ++i) ++gmult[size_t(qb) * kKvMax + c[i]];
            } else {  // every query of a block has the same global tokens
                std::vector<uint8_t> gm(kKvMax, 0);
                for (uint32_t i = nw; i < n; ++i) ++gm[c[i]];
                if (!std::equal(gm.begin(), gm.end(), gmult.begin() + size_t(qb) * kKvMax))
                    config_error("queries of one block must share their global tokens");
            }
        }
    }
    if (wflag < 0) wflag = 0;
    if (gflag < 0) gflag = 0;
    // TMA box program: runs of consecutive frames, each covered exactly by boxes of <= 32
    // rows (one TMA op per run: the copy engine's per-op cost, not bytes, bounds small boxes;
    // no box reads a frame the block does not use)
    for (uint32_t qb = 0; qb < nqb && kv_ok; ++qb) {
        const uint16_t* fr = &kv_frames[size_t(qb) * kKvMax];
        const uint32_t R = kv_count[qb];
        uint32_t nb = 0, rows = 0;
        auto put = [&](uint32_t word) {
            if (nb >= uint32_t(kKvMax)) config_error("attention K/V load program too long");
            kv_box[size_t(qb) * kKvMax + nb++] = word;
        };
        for (uint32_t c0 = 0; c0 < R;) {
            uint32_t len = 1;
            while (c0 + len < R && fr[c0 + len] == fr[c0] + len) ++len;
            if (gather4 && len == 1) {
                // a run of isolated frames (sampled globals outside the window band):
                // four per row-gather while four remain, as 3 words
                uint32_t n1 = 1;
                while (c0 + n1 < R && (c0 + n1 + 1 >= R || fr[c0 + n1 + 1] != fr[c0 + n1] + 1)) ++n1;
                while (n1 >= 4) {
                    put(uint32_t(fr[c0]) | c0 << 16 | uint32_t(kBoxGather4) << 24);
                    put(uint32_t(fr[c0 + 1]) | uint32_t(fr[c0 + 2]) << 16);
                    put(uint32_t(fr[c0 + 3]));
                    rows += 4;
                    c0 += 4;
                    n1 -= 4;
                }
                if (n1 == 0) continue;
                len = 1;
            }
            uint32_t at = 0;
            while (at < len) {
                const uint32_t h = std::min<uint32_t>(len - at, uint32_t(kBoxKinds));
                put(uint32_t(fr[c0 + at]) | (c0 + at) << 16 | (h - 1) << 24);
                rows += h;
                at += h;
            }
            c0 += len;
        }
        kv_nbox[qb] = uint16_t(nb);
        kv_load_rows[qb] = uint16_t(rows);
    }
}

size_t HostTokens::blob_bytes() const {
    return kv_box.size() * 4 + rows.size() * 2 + biased.size() + col.size() + count.size() * 2 +
           kv_frames.size() * 2 + kv_count.size() * 2 + kv_nbox.size() * 2 + kv_load_rows.size() * 2 +
           wlo.size() + whi.size() + gmult.size() + 64;
}

void HostTokens::pack(uint8_t* dst) const {
    size_t o = 0;
    auto put = [&](const void* src, size_t n) {
        if (n) std::memcpy(dst + o, src, n);
        o += n;
    };
    put(kv_box.data(), kv_box.size() * 4);
    put(rows.data(), rows.size() * 2);
    put(kv_frames.data(), kv_frames.size() * 2);
    put(kv_nbox.data(), kv_nbox.size() * 2);
    put(kv_load_rows.data(), kv_load_rows.size() * 2);
    put(count.data(), count.size() * 2);
    put(kv_count.data(), kv_count.size() * 2);
    put(biased.data(), biased.size());
    put(col.data(), col.size());
    put(wlo.data(), wlo.size());
    put(whi.data(), whi.size());
    put(gmult.data(), gmult.size());
}

TokenTable HostTokens::view(const uint8_t* base) const {
    TokenTable t{};
    size_t o = 0;
    t.kv_box = reinterpret_cast<const uint32_t*>(base + o);
    o += kv_box.size() * 4;
    t.rows = reinterpret_cast<const uint16_t*>(base + o);
    o += rows.size() * 2;
    t.kv_frames = reinterpret_cast<const uint16_t*>(base + o);
    o += kv_frames.size() * 2;
    t.kv_nbox = reinterpret_cast<const uint16_t*>(base + o);
    o += kv_nbox.size() * 2;
    t.kv_load_rows = reinterpret_cast<const uint16_t*>(base + o);
    o += kv_load_rows.size() * 2;
    t.count = reinterpret_cast<const uint16_t*>(base + o);
    o += count.size() * 2;
    t.kv_count = reinterpret_cast<const uint16_t*>(base + o);
    o += kv_count.size() * 2;
    t.biased = base + o;
    o += biased.size();
    t.col = base + o;
    o += col.size();
    t.wlo = base + o;
    o += wlo.size();
    t.whi = base + o;
    o += whi.size();
    t.gmult = base + o;
    t.wflag = wflag;
    t.gflag = gflag;
    t.kv_ok = kv_ok ? 1 : 0;
    t.max_kv = 0;
    for (uint16_t c : kv_count) t.max_kv = std::max<int>(t.max_kv, c);
    return t;
}

// ---------------------------------------------------------------------------
// Engine layout

namespace {
uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
}  // namespace

Layout::Layout(const vinf_engine_desc& desc) : d(desc) {
    if (d.height == 0 || d.width == 0 || d.channels == 0) shape_error("zero tensor dimension");
    if (d.taps == 0 || d.taps % 2 == 0) config_error("conv taps must be odd and >= 1");
    if (d.groups == 0 || d.channels % d.groups != 0)
        config_error("norm groups must divide channels: groups=" + std::to_string(d.groups) +
                     " channels=" + std::to_string(d.channels));
    if (d.heads == 0 || d.channels % d.heads != 0) config_error("heads must divide channels");

    if (d.blocks == 0) config_error("model needs at least one block");
    if (!(d.epsilon > 0.0f)) config_error("group norm epsilon must be > 0");
    if (d.channels % 8 != 0)
        shape_error("the clip engine needs channels % 8 == 0 (16-byte TMA rows)");
    if ((d.channels / d.heads) % 8 != 0)
        config_error("attention head dim (channels / heads) must be a multiple of 8");
    if (d.uneven) {
        if (d.workers == 0 || d.frames < d.workers) config_error("uneven clips need frames >= workers >= 1");
    } else {
        make_plan(d.frames, d.workers);  // the reference's even split (clip_parallel.cpp:56-59)
    }
    if (d.worker >= d.workers) range_error("worker index out of range");
    f_clip = clip_start(d.worker + 1) - clip_start(d.worker);
    uint32_t min_clip = f_clip;
    for (uint32_t w = 0; w < d.workers; ++w)
        min_clip = std::min(min_clip, clip_start(w + 1) - clip_start(w));
    hw = d.height * d.width;
    hc = (d.taps - 1) / 2;
    ha = d.n_local / 2;
    // pipeline.cpp:131-143
    if (hc > min_clip)
        config_error("conv halo exceeds clip: (taps-1)/2 = " + std::to_string(hc) +
                     " > frames/workers = " + std::to_string(min_clip));
    if (ha > min_clip)
        config_error("attention halo exceeds clip: n_local/2 = " + std::to_string(ha) +
                     " > frames/workers = " + std::to_string(min_clip));
    if (d.n_local + 1 + d.n_global > uint32_t(kMaxTokens))
        config_error("n_local + 1 + n_global exceeds " + std::to_string(kMaxTokens));
    gset = build_global_index_set(d.frames, d.n_global);
    start = clip_start(d.worker);
    f32 = d.dtype == VINF_F32;
    es = f32 ? 4 : 2;
    E = uint64_t(hw) * d.channels;
    scale = d.scale > 0.0f ? d.scale : 1.0f / std::sqrt(float(d.channels / d.heads));

    npre_c = d.worker > 0 ? hc : 0;
    npost_c = d.worker + 1 < d.workers ? hc : 0;
    npre_a = d.worker > 0 ? ha : 0;
    npost_a = d.worker + 1 < d.workers ? ha : 0;

    // Global frames: local (inside this worker's synchronized window) or remote.
    auto ext_lo = [&](uint32_t w) { return clip_start(w) - (w > 0 ? ha : 0); };
    auto ext_hi = [&](uint32_t w) { return clip_start(w + 1) + (w + 1 < d.workers ? ha : 0); };
    g_frame.assign(d.n_global, 0);
    n_remote = 0;
    for (uint32_t j = 0; j < d.n_global; ++j) {
        const uint32_t g = gset[j];
        if (g >= ext_lo(d.worker) && g < ext_hi(d.worker))
            g_frame[j] = ha + (g - start);  // may sit in a halo slot (g < start)
        else
            g_frame[j] = 2 * ha + f_clip + n_remote++;
    }
    cf = hc + f_clip + hc;
    null_frame = 2 * ha + f_clip + n_remote;
    af = null_frame + 1;
    if (af > 0xFFFFu) config_error("attention buffer exceeds 65535 frames (16-bit token rows)");

    // Token lists (clip_parallel.cpp:285-305): window first, then the global set. With
    // the attention sync ablated the reference attends zero stand-ins for every global
    // token (clip_parallel.cpp:118-121, 315-318), own members included: tables 2, 3 point
    // all global tokens at the never-written null frame.
    for (int b = 0; b < 4; ++b) {
        tok[b].resize(f_clip);
        for (uint32_t a = 0; a < f_clip; ++a) {
            for (uint32_t g : build_local_window(start + a, d.frames, d.n_local))
                tok[b].push(a, ha + g - start, (b & 1) == 0);
            for (uint32_t j = 0; j < d.n_global; ++j)
                tok[b].push(a, b >= 2 ? null_frame : g_frame[j], (b & 1) == 1, true);
        }
        tok[b].finalize((d.channels / d.heads) % 64 == 0);
        if (!tok[b].kv_ok) config_error("a query block touches more than 192 distinct frames");
    }

    // Workspace regions.
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) {
        const uint64_t o = off;
        off = align_up(off + bytes, 1024);
        return o;
    };
    const uint64_t clip = uint64_t(f_clip) * E;
    off_x = take(clip * es);
    off_y = take(clip * es);
    off_tmp = d.blocks > 1 ? take(clip * es) : off_y;  // intermediate block outputs
    off_u0 = take(uint64_t(cf) * E * 2);  // bf16 plane (bf16 mode) / hi plane (f32 mode)
    off_u0lo = f32 ? take(uint64_t(cf) * E * 2) : 0;
    off_u0f = f32 ? take(clip * 4) : 0;
    off_u1 = take(clip * es);
    off_u2 = take(uint64_t(af) * E * 2);
    off_u2lo = f32 ? take(uint64_t(af) * E * 2) : 0;
    off_u2f = f32 ? take(clip * 4) : 0;
    off_qkv = take(uint64_t(af) * E * 3 * es);
    off_ctx = take(clip * 2);
    off_ctxlo = f32 ? take(clip * 2) : 0;
    off_sums = take(sizeof(double) * 2 * d.groups);
    if (!f32) {
        off_wfold = take(uint64_t(3) * d.channels * d.channels * 2);
        off_gnaff = take(sizeof(float) * 5 * d.channels);
    }
    off_stats = take(sizeof(double) * 2 * d.groups);
    scratch_elems = std::max<uint64_t>(uint64_t(kScratchBlocks) * d.groups,
                                       uint64_t(256) * 2 * d.channels);  // colpart segments
    off_scratch = take(sizeof(double) * scratch_elems);
    // column-statistic partial rows: 4 per 128-row tile bounds both layouts (gemm_colpart_rows)
    off_colstats = take(sizeof(float) * 2 * d.channels * 4 * ((uint64_t(f_clip) * hw + 127) / 128));
    for (int b = 0; b < 4; ++b) off_tok[b] = take(tok[b].blob_bytes());
    total = off;

    build_exchanges();
}

void Layout::build_exchanges() {
    const uint32_t i = d.worker, n = d.workers;
    const uint64_t fb = E * 2;  // one frame of one bf16 plane
    const int planes = f32 ? 2 : 1;
    auto plane_off = [&](bool conv, int p) {
        return conv ? (p == 0 ? off_u0 : off_u0lo) : (p == 0 ? off_u2 : off_u2lo);
    };
    auto halos = [&](std::vector<vinf_xfer>& xs, bool conv, uint32_t h, uint32_t stage) {
        if (h == 0 || n == 1) return;
        const uint32_t hslot = conv ? hc : ha;  // halo slot width in the buffer
        for (int p = 0; p < planes; ++p) {
            const uint64_t base = plane_off(conv, p);
            // tag: stage * 1000 + direction * 10 + plane (direction 0 = i -> i+1)
            if (i + 1 < n) {
                // last h own frames -> next worker's pre slot; next's first h -> our post slot
                xs.push_back({i + 1, 1, stage * 1000 + 0 * 10 + uint32_t(p), 0,
                              base + uint64_t(hslot + f_clip - h) * fb, uint64_t(h) * fb});
                xs.push_back({i + 1, 0, stage * 1000 + 1 * 10 + uint32_t(p), 0,
                              base + uint64_t(hslot + f_clip) * fb, uint64_t(h) * fb});
            }
            if (i > 0) {
                xs.push_back({i - 1, 0, stage * 1000 + 0 * 10 + uint32_t(p), 0,
                              base + uint64_t(hslot - h) * fb, uint64_t(h) * fb});
                xs.push_back({i - 1, 1, stage * 1000 + 1 * 10 + uint32_t(p), 0,
                              base + uint64_t(hslot) * fb, uint64_t(h) * fb});
            }
        }
    };
    xconv.clear();
    xattn.clear();
    halos(xconv, true, hc, 1);
    halos(xattn, false, ha, 2);
    if (n > 1 && d.n_global > 0) {
        // Remote global frames: the owner sends each of its members to every worker for
        // which the frame lies outside the synchronized window (T1, clip_parallel.cpp:114-148,
        // minus frames the receiver already holds).
        auto lo_of = [&](uint32_t w) { return clip_start(w) - (w > 0 ? ha : 0); };
        auto hi_of = [&](uint32_t w) { return clip_start(w + 1) + (w + 1 < n ? ha : 0); };
        std::vector<uint32_t> slot_count(n, 0);
        for (uint32_t j = 0; j < d.n_global; ++j) {
            const uint32_t g = gset[j];
            uint32_t owner = 0;
            while (owner + 1 < n && clip_start(owner + 1) <= g) ++owner;
            for (uint32_t r = 0; r < n; ++r) {
                if (g >= lo_of(r) && g < hi_of(r)) continue;  // local to r
                const uint32_t slot = slot_count[r]++;
                if (r == owner) continue;  // cannot happen (own frames are local)
                for (int p = 0; p < planes; ++p) {
                    const uint32_t tag = 3000 + j * 4 + uint32_t(p);
                    const uint64_t base = plane_off(false, p);
                    if (owner == i)
                        xattn.push_back({r, 1, tag, 0, base + uint64_t(ha + g - start) * fb, fb});
                    if (r == i)
                        xattn.push_back(
                            {owner, 0, tag, 0, base + uint64_t(2 * ha + f_clip + slot) * fb, fb});
                }
            }
        }
    }
}

}  // namespace vinf
