// workspace.h -- carving of the caller-provided device workspace.
#pragma once
#include <cstddef>
#include <cstdint>

#include "kernels.h"
#include "tfla/tfla.h"

namespace tfla_host {

struct WsPlan {
    size_t b, ib, mc, ab, bb, dinv, gbar, gsum, amax;  // gate vectors
    size_t gtmp;                                       // K0: f64 per-position b, a, ib, m_intra (chunk pass -> finalize)
    size_t n_states;                                   // fwd: internal n (exp)
    size_t u_part;                                     // fwd: K1 n increments per x tile
    size_t saved;                                      // bf16 C_0..C_{NC-1}
    size_t dstates;                                    // bwd: bf16 dC_1..dC_NC
    size_t dg_part, dbq, da, colsum;                   // bwd partials
    size_t iq, dg;                                     // bwd (fused): w q.(C dh) per token, d_g
    size_t total;
    int ntile, n_ptile, n_xtile;
    int scan_ntile, n_scan_tiles;  // state-scan (K1/K3) column tile and tiles per chunk
};

// K1 / K3 column tile: 64 -> two CTAs per SM (state_scan.cu)
constexpr int kScanNTile = 64;

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

inline int pick_ntile(const tfla_dims& d, const tfla_blocks* blocks) {
    if (blocks && (blocks->b_dhv == 64 || blocks->b_dhv == 128) && d.d_hv % blocks->b_dhv == 0)
        return static_cast<int>(blocks->b_dhv);
    return d.d_hv % 128 == 0 ? 128 : 64;
}

inline WsPlan plan_workspace(const tfla_dims& d, int pass, int ntile) {
    WsPlan p{};
    const size_t BH = static_cast<size_t>(d.n_batch) * d.n_head;
    const size_t T = d.T, NC = d.T / d.L;
    const size_t BT = BH * T;
    p.ntile = ntile;
    p.n_xtile = static_cast<int>(d.d_hv / ntile);
    p.n_ptile = static_cast<int>((d.d_qk + 127) / 128);
    p.scan_ntile = kScanNTile;
    // partial buffers sized for the narrowest (32-column) scan tiles
    p.n_scan_tiles = p.n_ptile * static_cast<int>((d.d_hv + 31) / 32);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += align_up(bytes);
        return o;
    };
    p.b = take(BT * 4);
    p.ib = take(BT * 4);
    p.mc = take(BT * 4);
    p.ab = take(BT * 4);
    p.bb = take(BT * 4);
    p.dinv = take(BT * 4);
    p.gbar = take(BH * NC * 4);
    p.gsum = take(BH * NC * 8);
    p.amax = take(BH * NC * 8);
    p.gtmp = take(BT * 4 * 8);
    p.n_states = take(BH * (NC + 1) * d.d_qk * 4);
    p.u_part = take(BH * NC * ((d.d_hv + 31) / 32) * d.d_qk * 4);
    p.saved = take(BH * NC * d.d_qk * d.d_hv * 2);
    if (pass == 1) {
        p.dstates = take(BH * NC * d.d_qk * d.d_hv * 2);
        p.dg_part = take(BH * NC * p.n_scan_tiles * 4);
        p.dbq = take(static_cast<size_t>(p.n_ptile) * BT * 4);
        p.da = take(static_cast<size_t>(p.n_ptile) * BT * 4);
        p.colsum = take(BT * 4);
        p.iq = take(BT * 4);
        p.dg = take(BH * NC * 4);
    }
    p.total = off;
    return p;
}

// Stabiliser audit counters of the current device (nullptr when disabled).
tfla_k::StabCounters* stab_counters();

inline tfla_k::GateWS gate_ws(const WsPlan& p, void* ws) {
    uint8_t* w = static_cast<uint8_t*>(ws);
    tfla_k::GateWS g;
    g.b = reinterpret_cast<float*>(w + p.b);
    g.ib = reinterpret_cast<float*>(w + p.ib);
    g.mc = reinterpret_cast<float*>(w + p.mc);
    g.ab = reinterpret_cast<float*>(w + p.ab);
    g.bb = reinterpret_cast<float*>(w + p.bb);
    g.dinv = reinterpret_cast<float*>(w + p.dinv);
    g.gbar = reinterpret_cast<float*>(w + p.gbar);
    g.gsum = reinterpret_cast<double*>(w + p.gsum);
    g.amax = reinterpret_cast<double*>(w + p.amax);
    g.gtmp = reinterpret_cast<double*>(w + p.gtmp);
    g.stab = stab_counters();
    return g;
}

inline tfla_k::Geom geom_of(const tfla_dims& d) {
    tfla_k::Geom g;
    g.BH = static_cast<int>(d.n_batch * d.n_head);
    g.T = static_cast<int>(d.T);
    g.L = static_cast<int>(d.L);
    g.NC = static_cast<int>(d.T / d.L);
    g.dqk = static_cast<int>(d.d_qk);
    g.dhv = static_cast<int>(d.d_hv);
    return g;
}

}  // namespace tfla_host
