// Tiling of the i<j molecule-pair triangle used by the partner-search kernel
// and the multi-GPU shard plan.  Molecules are grouped in 32-molecule tiles
// (one warp-ballot word per tile pair and row); `st` x `st` tiles form a
// super-tile processed by one CTA of `st` warps.  Larger super-tiles make the
// bit-matrix stores full 32-byte sectors; small systems use small super-tiles
// so the grid still covers the 148 SMs.
#pragma once

namespace b2md {

struct SearchGeometry {
  int n = 0;        // molecules
  int n_tiles = 0;  // ceil(n / 32)
  int st = 1;       // tiles per super-tile side
  int n_super = 0;  // super-tile rows = ceil(n_tiles / st)
  int n_pad = 0;    // n_super * st * 32 (rows of the bit matrix)
  int words = 0;    // 32-bit words per bit-matrix row = n_super * st
};

inline SearchGeometry search_geometry(int n) {
  SearchGeometry g;
  g.n = n;
  g.n_tiles = (n + 31) / 32;
  g.st = n >= 8192 ? 8 : (n >= 4096 ? 4 : (n >= 1536 ? 2 : 1));
  g.n_super = (g.n_tiles + g.st - 1) / g.st;
  g.words = g.n_super * g.st;
  g.n_pad = g.words * 32;
  return g;
}

}  // namespace b2md
