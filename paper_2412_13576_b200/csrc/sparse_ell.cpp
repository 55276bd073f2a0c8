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
    for (int e = 0;; ++e) {
        bool any = false;
        for (int L = 0; L < 32; ++L) any |= ln[L].pos < mine[L].size();
        if (!any) break;
        uint32_t used = 0;
        uint32_t slot[32];
        bool later[32];
        for (int k = 0; k < 32; ++k) {   // lanes with real entries pick first (rotating priority)
            const int L = (e + k) & 31;
            Lane& s = ln[L];
            later[L] = s.pos >= mine[L].size() || s.rem.empty();
            if (later[L]) continue;
            size_t pick = 0;
            bool got = false;
            for (size_t c = 0; c < s.rem.size(); ++c)
                if (!(used & (1u << (s.rem[c].first & 31)))) {
                    pick = c;
                    got = true;
                    break;
                }
            if (!got) ++S.conflicts;
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
