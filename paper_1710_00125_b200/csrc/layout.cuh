// Device workspace layout of rcp_factor (shared by the factor driver and the multi-GPU
// Schur workers, which address rank 0's workspace through a CUDA IPC mapping).
#pragma once
#include <algorithm>
#include <cstddef>
#include <cstdint>

#include "../../include/rcp_b200.h"
#include "dist.cuh"
#include "panel.cuh"
#include "rcp_common.cuh"

namespace rcp {

constexpr size_t kAlign = 256;

inline size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

struct Layout {
  size_t A0, A1, Lbuf, lorig, W, Lneg, Wg, B0, B1, qscr, Y, L11, omega, phys, lop, pol, perm0, perm1, poso, snap, tstamp, flags, xrec, qrec,
      qcol, sdec, qdec, state, scal, desc, plog, dist, total;
  int64_t rows_pad, snap_cap;
  int tpad;
};

inline Layout make_layout(int64_t n, const rcp_config& c) {
  Layout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  const size_t nn = (size_t)n * (size_t)n;
  const int P = c.p;
  L.tpad = ((c.b + 2 + 15) / 16) * 16;
  L.rows_pad = ((n + 127) / 128) * 128;
  int64_t per_panel_min = std::max<int64_t>(1, (int64_t)c.b - 1);
  int64_t max_panels = n / per_panel_min + 2;
  L.snap_cap = std::min<int64_t>(max_panels * n, n * (n + 1) / 2 + n);
  L.A0 = take(nn * 8);
  L.A1 = take(nn * 8);
  L.Lbuf = take(nn * 8);
  L.lorig = take(nn * 8);  // L rows by original index, filled panel by panel (final-row assembly)
  L.W = take((size_t)n * (c.b + 2) * 8);
  L.Lneg = take((size_t)L.rows_pad * L.tpad * 8);
  L.Wg = take((size_t)L.rows_pad * L.tpad * 8);
  L.B0 = take((size_t)P * n * 8);
  L.B1 = take((size_t)P * n * 8);
  L.qscr = take((size_t)P * n * 8);
  L.Y = take((size_t)P * L.tpad * 8);
  L.L11 = take((size_t)L.tpad * L.tpad * 8);
  L.omega = take((size_t)P * n * 8);
  L.phys = take((size_t)n * 4);
  L.lop = take((size_t)n * 4);
  L.pol = take((size_t)n * 4);
  L.perm0 = take((size_t)n * 4);
  L.perm1 = take((size_t)n * 4);
  L.poso = take((size_t)n * 4);
  L.snap = take((size_t)L.snap_cap * 4);
  L.tstamp = take(8 * 4 * (size_t)(n + 2));  // per panel: panel start/end, Schur start/end (ns)
  L.flags = take(0);
  L.xrec = take(8 * 2 * kMaxSMs * (size_t)kXWords);
  L.qrec = take(8 * 2 * kMaxSMs * (size_t)kQWords);
  L.qcol = take(8 * 2 * kMaxSMs * qcol_stride(P));
  L.sdec = take(8 * 2 * kMaxSMs * (size_t)kMWords);  // per-CTA decision mailboxes (SBKP)
  L.qdec = take(8 * 2 * kMaxSMs * (size_t)kMWords);  // per-CTA decision mailboxes (QRCP, q = 1 pivot)
  L.state = take(sizeof(PanelState));
  L.scal = take(64);
  L.desc = take(2 * sizeof(PanelDesc));
  L.plog = take((size_t)(n + 2) * sizeof(PanelLog));
  L.dist = take(sizeof(DistShared));
  L.total = off;
  return L;
}


}  // namespace rcp
