// mtjump.h — std::mt19937_64 jump-ahead polynomials (host side, mtjump.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace hg {

constexpr int kMtPolyWords = 312;  // 19968 bits >= deg P = 19937

int mt_charpoly_degree();
// out = x^J mod P (kMtPolyWords words), cached per J.
void mt_jump_poly(uint64_t J, uint64_t* out);
// polys[c - c_first] = x^(offset0 + c*len - 1) mod P for c = c_first .. chunks-1,
// c_first = (offset0 == 0 ? 1 : 0): the polynomials that move a fresh engine to
// draw offset0 + c*len (applied by k_mt_jump).  Cached per (offset0, len, chunks).
const std::vector<uint64_t>& mt_chunk_polys(uint64_t offset0, uint64_t len, int chunks);
// Set-bit offsets of each polynomial per 312-bit block (the form k_mt_jump
// consumes): poly k's bits in block q are 312q + pool[starts[65k + q] ..
// starts[65k + q + 1]).
void mt_poly_offsets(const uint64_t* polys, int npolys, std::vector<int>& starts, std::vector<uint16_t>& pool);
// Host reference: the raw-word window x_J .. x_{J+311} of the engine seeded with
// engine_seed, i.e. the saved state (pos = 312) after J draws.
void mt_jump_state_host(uint64_t engine_seed, uint64_t J, uint64_t* window);

}  // namespace hg
