// Host construction of the lane-major ELL schedules the SIMT descent kernel runs (k_descent_simt.cu).
//
// A sparse product  out[o] = sum_{e in list o} val_e * x[idx_e]  (o = rows of B for the forward y = B z,
// columns of B for the backward Γ = B^T s) is split over the 32 lanes of a warp. Lists longer than a chunk
// size are cut into pieces; pieces go to lanes longest-first onto the least-loaded lane, and lane L walks its
// pieces in slots e = 0, 1, ... reading word [e * 32 + L]:
//     bits  2-15  idx  (the gathered x index; the low 16 bits are the byte offset 4 * idx)
//     bit   0     END  (the lane's current piece is complete after this word)
//     bits 16-31  val  (bf16 of the B entry: exact for |B| <= 256; 0 for PAD words)
// At END the lane appends its sum to its result queue res[k * 32 + L] (k-th piece). A post pass stores
// res[q * 32 + L] to owned[q * 32 + L] (an output >= 0; -1 for the pieces of split outputs), and a fixup pass
// sums the pieces of each split output in piece order. So a warp reads one 128-byte line of words per slot and
// every sum has a fixed order (deterministic across runs). Within a piece the summation order is free, and the
// builder uses that freedom: in every slot it gives each lane, where it can, an entry whose gathered index falls
// in a shared-memory bank (idx mod 32) no other lane of that slot uses, so the gather x[idx] is one
// conflict-free wavefront. PAD words (finished lanes, and the one word of an empty piece) gather an unused
// bank with val 0.
#pragma once
#include <cstdint>
#include <vector>

namespace maple {

struct EllSchedule {
    int slots = 0;                 // L: words per lane
    int max_pieces = 0;            // Q: the most pieces any lane owns
    std::vector<uint32_t> words;   // slots * 32
    std::vector<int32_t> owned;    // Q * 32: output of lane L's q-th piece (>= 0), -1 (split output / unused)
    std::vector<int32_t> fixup;    // triples (output, first, count) into fixpos, ascending output
    std::vector<int32_t> fixpos;   // queue positions q * 32 + L of each split output's pieces, in order
    int conflicts = 0;             // slot-lanes that could not get a free bank
};

constexpr uint32_t kEllEnd = 1u;
constexpr int kEllMaxIndex = 16383;

// lists[o] = (idx, val) entries of output o (idx <= kEllMaxIndex, |val| <= 256); gather_limit = size of the
// gathered array (PAD indices < it); chunk = max piece length (0: never split, e.g. Adam-owned coordinates).
EllSchedule build_ell(const std::vector<std::vector<std::pair<int, int>>>& lists, int gather_limit, int chunk);

}  // namespace maple
