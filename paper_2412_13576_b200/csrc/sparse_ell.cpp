#include "sparse_ell.h"

#include <algorithm>
#include <cstring>
#include <numeric>

namespace maple {

EllSchedule build_ell(const std::vector<std::vector<std::pair<int, int>>>& lists, int gather_limit, int chunk) {
    const int no = (int)lists.size();
    EllSchedule S;
    struct Piece {
        int out;    // output index
        int part;   // index of its split output, or -1 for a whole list
        std::vector<std::pair<int, int>> ent;
    };
    std::vector<Piece> pieces;
    std::vector<std::vector<int>> split;   // per split output: its piece indices, in order
    for (int o = 0; o < no; ++o) {
        const auto& l = lists[o];
        if (chunk <= 0 || (int)l.size() <= chunk) {
            pieces.push_back({o, -1, l});
            continue;
        }
        split.emplace_back();
        for (size_t b = 0; b < l.size(); b += (size_t)chunk) {
            split.back().push_back((int)pieces.size());
            pieces.push_back({o, (int)split.size() - 1, std::vector<std::pair<int, int>>(
                                  l.begin() + (long)b, l.begin() + (long)std::min(l.size(), b + (size_t)chunk))});
        }
    }
    // longest piece first onto the least-loaded lane (an empty list still costs its one word)
    std::vector<int> ord(pieces.size());
    std::iota(ord.begin(), ord.end(), 0);
    auto cost = [&](int p) { return std::max<int>(1, (int)pieces[p].ent.size()); };
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return cost(a) > cost(b); });
    std::vector<std::vector<int>> mine(32);
    std::vector<int> load(32, 0);
    for (int p : ord) {
        const int L = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        mine[L].push_back(p);
        load[L] += cost(p);
    }
    for (auto& v : mine) {
        std::sort(v.begin(), v.end());   // a lane walks its pieces in output order
        S.max_pieces = std::max(S.max_pieces, (int)v.size());
    }
    S.owned.assign((size_t)std::max(S.max_pieces, 1) * 32, -1);
    std::vector<int> pos(pieces.size(), -1);
    for (int L = 0; L < 32; ++L)
        for (size_t q = 0; q < mine[L].size(); ++q) {
            const Piece& pc = pieces[mine[L][q]];
            pos[mine[L][q]] = (int)q * 32 + L;
            if (pc.part < 0) S.owned[q * 32 + L] = pc.out;
        }
    for (const auto& sp : split) {
        S.fixup.insert(S.fixup.end(), {pieces[sp[0]].out, (int)S.fixpos.size(), (int)sp.size()});
        for (int p : sp) S.fixpos.push_back(pos[p]);
    }

    struct Lane {
        size_t pos = 0;                        // current piece (index into mine[L])
        std::vector<std::pair<int, int>> rem;  // its remaining entries
    };
    std::vector<Lane> ln(32);
    for (int L = 0; L < 32; ++L)
        if (!mine[L].empty()) ln[L].rem = pieces[mine[L][0]].ent;
    auto word = [](int idx, int val, bool end) {   // bf16 of a small integer: the top half of its fp32
        const float f = (float)val;
        uint32_t b;
        std::memcpy(&b, &f, 4);
        return ((uint32_t)idx << 2) | (b & 0xFFFF0000u) | (end ? kEllEnd : 0u);
    };
    auto free_bank = [&](uint32_t used) {
        int b = 0;
        while (b < 32 && ((used >> b) & 1u)) ++b;
        return (b < 32 && b < gather_limit) ? b : 0;
    };
    // Per slot: a maximum matching of the lanes that hold real entries to shared-memory banks (lane L may take
    // bank b if an entry of its current piece gathers from bank b; Kuhn's augmenting paths, lanes with the
    // fewest options first), so as many lanes as possible gather conflict-free. A lane left unmatched takes the
    // entry whose bank is least used in the slot (the gather then costs two wavefronts; keep it at two).
    for (int e = 0;; ++e) {
        bool any = false;
        for (int L = 0; L < 32; ++L) any |= ln[L].pos < mine[L].size();
        if (!any) break;
        uint32_t used = 0;
        uint32_t slot[32];
        bool later[32];
        uint32_t opts[32];
        int order[32], nact = 0;
        for (int L = 0; L < 32; ++L) {
            Lane& s = ln[L];
            later[L] = s.pos >= mine[L].size() || s.rem.empty();
            opts[L] = 0;
            if (later[L]) continue;
            for (const auto& en : s.rem) opts[L] |= 1u << (en.first & 31);
            order[nact++] = L;
        }
        std::stable_sort(order, order + nact, [&](int a, int b) {
            const int pa = __builtin_popcount(opts[a]), pb = __builtin_popcount(opts[b]);
            return pa != pb ? pa < pb : ((a - e) & 31) < ((b - e) & 31);
        });
        int bank_of[32], lane_of[32];
        for (int k = 0; k < 32; ++k) bank_of[k] = lane_of[k] = -1;
        for (int k = 0; k < nact; ++k) {
            const int L0 = order[k];
            uint32_t seen = 0;
            // iterative DFS for an augmenting path from lane L0
            struct Fr { int lane; uint32_t left; };
            Fr st[33];
            int sp = 0;
            st[sp++] = {L0, opts[L0]};
            int path_bank[33];
            bool found = false;
            while (sp > 0 && !found) {
                Fr& fr = st[sp - 1];
                const uint32_t cand = fr.left & ~seen;
                if (!cand) { --sp; continue; }
                const int b = __builtin_ctz(cand);
                fr.left &= ~(1u << b);
                seen |= 1u << b;
                path_bank[sp - 1] = b;
                if (lane_of[b] < 0) { found = true; break; }
                st[sp++] = {lane_of[b], opts[lane_of[b]]};
            }
            if (found)
                for (int q = sp - 1; q >= 0; --q) {   // flip the path: lane st[q] takes bank path_bank[q]
                    const int L = st[q].lane, b = path_bank[q];
                    bank_of[L] = b;
                    lane_of[b] = L;
                }
        }
        int cnt[32] = {0};
        for (int L = 0; L < 32; ++L)
            if (!later[L] && bank_of[L] >= 0) cnt[bank_of[L]]++;
        for (int k = 0; k < nact; ++k) {
            const int L = order[k];
            Lane& s = ln[L];
            size_t pick = 0;
            if (bank_of[L] >= 0) {
                for (size_t c = 0; c < s.rem.size(); ++c)
                    if ((s.rem[c].first & 31) == bank_of[L]) { pick = c; break; }
            } else {
                ++S.conflicts;
                int best = 1 << 30;
                for (size_t c = 0; c < s.rem.size(); ++c) {
                    const int b = s.rem[c].first & 31;
                    if (cnt[b] < best) { best = cnt[b]; pick = c; }
                }
                cnt[s.rem[pick].first & 31]++;
            }
            const auto ent = s.rem[pick];
            s.rem.erase(s.rem.begin() + (long)pick);
            used |= 1u << (ent.first & 31);
            const bool end = s.rem.empty();
            slot[L] = word(ent.first, ent.second, end);
            if (end && ++s.pos < mine[L].size()) s.rem = pieces[mine[L][s.pos]].ent;
        }
        for (int L = 0; L < 32; ++L) {   // PAD words: finished lanes, and empty pieces (END, val 0)
            if (!later[L]) continue;
            Lane& s = ln[L];
            const int b = free_bank(used);
            used |= 1u << (b & 31);
            const bool end = s.pos < mine[L].size();   // an empty piece completes here
            slot[L] = word(b, 0, end);
            if (end && ++s.pos < mine[L].size()) s.rem = pieces[mine[L][s.pos]].ent;
        }
        S.words.insert(S.words.end(), slot, slot + 32);
        ++S.slots;
    }
    return S;
}

}  // namespace maple
