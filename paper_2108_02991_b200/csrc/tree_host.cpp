// tree_host.cpp -- host half of the treecode: octree over sorted Morton keys and the
// per-target-group interaction lists.
//
// Counterparts of the reference's build_tree (_treecode.py:77-170), dual_traverse
// (:173-244) and group_by_target (:247-262).  The reference builds a dual tree and
// interacts node pairs through M2L; here every target group (<= TR_GROUP consecutive
// targets in Morton order forming whole sibling subtrees of the target octree, tight
// bounding box computed on the GPU) walks the source octree and collects
//     near: particle ranges of leaves that fail the opening test, and
//     far : nodes that pass it -> their q^d Chebyshev proxies (or their particles when the
//           node holds no more particles than proxies),
// as (record offset, count) segments into [sorted sources | proxies].  All outputs are in
// a fixed order (BFS node order, depth-first child order), so results are deterministic.
// The production path runs the same traversal on the GPU (tree.cu traverse_kernel); this
// serial planner is its host reference -- tests require identical lists.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

#include "sparkling_b200.h"

namespace spk {
void set_error(const char* fmt, ...);
}

namespace {

struct Node {
    int64_t begin, end;
    int32_t first_child, n_child;
    int32_t level;
};

struct Box {
    float c[3], h[3];
    float r;  // half-diagonal
};

struct HostTree {
    int dims = 3;
    int64_t n = 0;
    std::vector<Node> nodes;
    std::vector<int32_t> leaves;
    std::vector<Box> box;
    // plan
    std::vector<int64_t> seg_off, seg_start;
    std::vector<int32_t> seg_count;
    std::vector<int32_t> slot_node;
    std::vector<float> slot_box;
    std::vector<int32_t> unit_slot;
    std::vector<int64_t> unit_begin, unit_end, slot_unit_off;
    int64_t near_pairs = 0, far_pairs = 0;
};

constexpr int64_t P2M_UNIT = 4096;  // particles per P2M work unit

Box make_box(const float* lohi, int dims) {
    Box b{};
    float r2 = 0.0f;
    for (int a = 0; a < 3; ++a) {
        const float lo = lohi[a], hi = lohi[3 + a];
        b.c[a] = 0.5f * (lo + hi);
        b.h[a] = a < dims ? 0.5f * (hi - lo) : 0.0f;
        r2 += b.h[a] * b.h[a];
    }
    b.r = std::sqrt(r2);
    return b;
}

}  // namespace

extern "C" {

void* spk_tree_host_build(const uint64_t* keys, int64_t n, int dims, int64_t leaf_cap,
                          int min_level) {
    if (!(dims == 2 || dims == 3) || n <= 0 || leaf_cap < 1) {
        spk::set_error("tree build: bad arguments (n=%lld, dims=%d, leaf_cap=%lld)",
                       (long long)n, dims, (long long)leaf_cap);
        return nullptr;
    }
    HostTree* t = new (std::nothrow) HostTree;
    if (!t) {
        spk::set_error("tree build: out of host memory");
        return nullptr;
    }
    t->dims = dims;
    t->n = n;
    const int bits = dims == 3 ? 21 : 31;  // bits per axis (tree.cu keys_kernel)
    const int nc = 1 << dims;
    t->nodes.push_back(Node{0, n, -1, 0, 0});
    for (size_t i = 0; i < t->nodes.size(); ++i) {
        Node nd = t->nodes[i];
        const int64_t size = nd.end - nd.begin;
        const bool split = size > leaf_cap || (nd.level < min_level && size > 1);
        if (!split || nd.level >= bits) {
            t->leaves.push_back((int32_t)i);
            continue;
        }
        const int shift = dims * (bits - nd.level - 1);
        const uint64_t prefix = keys[nd.begin] >> (shift + dims);
        int64_t lo = nd.begin;
        const int32_t first = (int32_t)t->nodes.size();
        int32_t cnt = 0;
        for (int c = 0; c < nc; ++c) {
            int64_t hi = nd.end;
            if (c + 1 < nc) {
                const uint64_t bound = ((prefix << dims) | (uint64_t)(c + 1)) << shift;
                hi = std::lower_bound(keys + lo, keys + nd.end, bound) - keys;
            }
            if (hi > lo) {
                t->nodes.push_back(Node{lo, hi, -1, 0, nd.level + 1});
                ++cnt;
            }
            lo = hi;
        }
        t->nodes[i].first_child = first;
        t->nodes[i].n_child = cnt;
    }
    t->box.assign(t->nodes.size(), Box{});
    return t;
}

void spk_tree_host_free(void* h) { delete static_cast<HostTree*>(h); }

/* BFS level offsets: nodes of level l are [off[l], off[l+1]).  Returns the number of
 * levels; off (may be NULL to count) receives levels + 1 entries. */
int64_t spk_tree_host_levels(const void* h, int64_t* off) {
    const HostTree* t = static_cast<const HostTree*>(h);
    const int32_t n_lv = t->nodes.back().level + 1;
    if (off) {
        int32_t l = 0;
        off[0] = 0;
        for (size_t i = 0; i < t->nodes.size(); ++i)
            while (t->nodes[i].level > l) off[++l] = (int64_t)i;
        off[n_lv] = (int64_t)t->nodes.size();
    }
    return n_lv;
}

/* Leaf node ids in BFS order. */
void spk_tree_host_leaf_nodes(const void* h, int32_t* ids) {
    const HostTree* t = static_cast<const HostTree*>(h);
    std::memcpy(ids, t->leaves.data(), t->leaves.size() * sizeof(int32_t));
}

/* counts[0] = nodes, counts[1] = leaves */
void spk_tree_host_sizes(const void* h, int64_t* counts) {
    const HostTree* t = static_cast<const HostTree*>(h);
    counts[0] = (int64_t)t->nodes.size();
    counts[1] = (int64_t)t->leaves.size();
}

/* Leaf record ranges (for the GPU box kernel) and the node table. */
void spk_tree_host_leaves(const void* h, int64_t* begin, int64_t* end) {
    const HostTree* t = static_cast<const HostTree*>(h);
    for (size_t k = 0; k < t->leaves.size(); ++k) {
        begin[k] = t->nodes[t->leaves[k]].begin;
        end[k] = t->nodes[t->leaves[k]].end;
    }
}

void spk_tree_host_nodes(const void* h, int64_t* begin, int64_t* end, int32_t* first_child,
                         int32_t* n_child, int32_t* level) {
    const HostTree* t = static_cast<const HostTree*>(h);
    for (size_t i = 0; i < t->nodes.size(); ++i) {
        const Node& nd = t->nodes[i];
        if (begin) begin[i] = nd.begin;
        if (end) end[i] = nd.end;
        if (first_child) first_child[i] = nd.first_child;
        if (n_child) n_child[i] = nd.n_child;
        if (level) level[i] = nd.level;
    }
}

/* Target groups of at most `cap` consecutive (sorted) particles that follow the octree:
 * consecutive sibling subtrees are packed while they fit, larger subtrees are split at
 * their children, oversized leaves (duplicate keys) are cut into chunks.  Returns the
 * number of groups; begin/end (may be NULL to count) receive the ranges. */
int64_t spk_tree_host_groups(const void* h, int64_t cap, int64_t* begin, int64_t* end) {
    const HostTree* t = static_cast<const HostTree*>(h);
    int64_t ng = 0;
    int64_t cur_b = -1, cur_e = -1;
    int32_t cur_parent = -2;
    auto emit = [&](int64_t b, int64_t e) {
        if (begin) begin[ng] = b, end[ng] = e;
        ++ng;
    };
    auto flush = [&]() {
        if (cur_b >= 0) emit(cur_b, cur_e);
        cur_b = cur_e = -1;
        cur_parent = -2;
    };
    std::vector<std::pair<int32_t, int32_t>> stack;  // (node, parent)
    stack.emplace_back(0, -1);
    while (!stack.empty()) {
        const auto [v, parent] = stack.back();
        stack.pop_back();
        const Node& nd = t->nodes[v];
        const int64_t cnt = nd.end - nd.begin;
        if (cnt <= cap && nd.n_child == 0) {
            // pack consecutive sibling leaves only: a group never spans two parents' cells
            if (cur_b >= 0 && parent == cur_parent && cur_e == nd.begin &&
                nd.end - cur_b <= cap) {
                cur_e = nd.end;
            } else {
                flush();
                cur_b = nd.begin, cur_e = nd.end, cur_parent = parent;
            }
        } else if (nd.n_child == 0) {
            flush();
            for (int64_t b = nd.begin; b < nd.end; b += cap) emit(b, std::min(nd.end, b + cap));
        } else {
            flush();
            for (int c = nd.n_child - 1; c >= 0; --c) stack.emplace_back(nd.first_child + c, v);
        }
    }
    flush();
    return ng;
}

/* Install the leaf boxes ([n_leaves][6] = min xyz, max xyz, spk_tree_boxes order) and
 * merge them up the tree. */
void spk_tree_host_set_leaf_boxes(void* h, const float* leaf_box) {
    HostTree* t = static_cast<HostTree*>(h);
    const size_t nn = t->nodes.size();
    std::vector<float> lohi(nn * 6);
    for (size_t k = 0; k < t->leaves.size(); ++k)
        std::memcpy(&lohi[(size_t)t->leaves[k] * 6], leaf_box + k * 6, 6 * sizeof(float));
    for (size_t ii = nn; ii-- > 0;) {  // children come after parents in BFS order
        const Node& nd = t->nodes[ii];
        if (nd.n_child == 0) continue;
        float* o = &lohi[ii * 6];
        for (int a = 0; a < 3; ++a) o[a] = INFINITY, o[3 + a] = -INFINITY;
        for (int c = 0; c < nd.n_child; ++c) {
            const float* cb = &lohi[(size_t)(nd.first_child + c) * 6];
            for (int a = 0; a < 3; ++a) {
                o[a] = std::min(o[a], cb[a]);
                o[3 + a] = std::max(o[3 + a], cb[3 + a]);
            }
        }
    }
    for (size_t i = 0; i < nn; ++i) t->box[i] = make_box(&lohi[i * 6], t->dims);
}

/* Interaction lists for n_groups target groups with boxes group_box [n_groups][6].
 * theta: opening parameter (far when r_t + r_s < theta * |c_t - c_s|); order: proxies per
 * axis; n_src: sorted source records before the proxy block.
 * counts[0..4] = segments, slots, units, near pairs (per target), far pairs (per target). */
static constexpr int32_t BREAK = INT32_MIN;  // raw list: no merge across this mark

int spk_tree_host_plan(void* h, int64_t n_groups, const float* group_box, double theta,
                       int order, int64_t n_src, int64_t* counts) {
    HostTree* t = static_cast<HostTree*>(h);
    const int dims = t->dims;
    const int64_t m = dims == 3 ? (int64_t)order * order * order : (int64_t)order * order;
    const int64_t nn = (int64_t)t->nodes.size();
    std::vector<std::vector<int32_t>> raw((size_t)n_groups);
    std::vector<char> is_proxy((size_t)nn, 0);
    const float th = (float)theta;

    for (int64_t g = 0; g < n_groups; ++g) {
        const Box tb = make_box(group_box + g * 6, dims);
        std::vector<int32_t>& out = raw[(size_t)g];
        int32_t stack[512];
        uint8_t depth[512];
        int sp = 0;
        depth[sp] = 0;
        stack[sp++] = 0;
        while (sp > 0) {
            const int32_t v = stack[--sp];
            const int dv = depth[sp];
            const Node& nd = t->nodes[v];
            // the device splits every walk into sub-walks at the tree's second level and
            // merges ranges only within one (tree.cu traverse_sub_kernel): break here too
            if (dv <= 2) out.push_back(BREAK);
            const Box& sb = t->box[v];
            float d2 = 0.0f;
            for (int a = 0; a < dims; ++a) {
                const float d = tb.c[a] - sb.c[a];
                d2 += d * d;
            }
            const float lhs = tb.r + sb.r;
            const bool far = lhs * lhs < th * th * d2;
            if (far) {
                if (nd.end - nd.begin > m) {
                    out.push_back(-1 - v);  // proxies
                    is_proxy[v] = 1;
                } else {
                    out.push_back(v);
                }
            } else if (nd.n_child == 0) {
                out.push_back(v);
            } else {
                if (sp + nd.n_child > 512) {
                    // cannot happen for depth <= 31 with <= 8 children per level
                    continue;
                }
                for (int c = nd.n_child - 1; c >= 0; --c) {
                    depth[sp] = (uint8_t)std::min(dv + 1, 255);
                    stack[sp++] = nd.first_child + c;
                }
            }
        }
    }

    // proxy slots in node order
    std::vector<int32_t> slot_of((size_t)nn, -1);
    t->slot_node.clear();
    for (int64_t v = 0; v < nn; ++v)
        if (is_proxy[v]) {
            slot_of[v] = (int32_t)t->slot_node.size();
            t->slot_node.push_back((int32_t)v);
        }
    const int64_t n_slots = (int64_t)t->slot_node.size();
    t->slot_box.assign((size_t)n_slots * 6, 0.0f);
    t->slot_unit_off.assign((size_t)n_slots + 1, 0);
    t->unit_slot.clear();
    t->unit_begin.clear();
    t->unit_end.clear();
    for (int64_t s = 0; s < n_slots; ++s) {
        const Node& nd = t->nodes[t->slot_node[s]];
        const Box& b = t->box[t->slot_node[s]];
        float hmax = 0.0f;
        for (int a = 0; a < dims; ++a) hmax = std::max(hmax, b.h[a]);
        for (int a = 0; a < 3; ++a) {
            t->slot_box[s * 6 + a] = b.c[a];
            // a degenerate axis (all particles share the coordinate) still needs h > 0
            t->slot_box[s * 6 + 3 + a] = a < dims ? std::max(b.h[a], 1e-6f * hmax + 1e-30f)
                                                  : 1.0f;
        }
        for (int64_t lo = nd.begin; lo < nd.end; lo += P2M_UNIT) {
            t->unit_slot.push_back((int32_t)s);
            t->unit_begin.push_back(lo);
            t->unit_end.push_back(std::min(nd.end, lo + P2M_UNIT));
        }
        t->slot_unit_off[s + 1] = (int64_t)t->unit_slot.size();
    }

    // raw lists -> merged (offset, count) segments
    std::vector<std::vector<std::pair<int64_t, int32_t>>> segs((size_t)n_groups);
    int64_t near_pairs = 0, far_pairs = 0;
    for (int64_t g = 0; g < n_groups; ++g) {
        auto& out = segs[(size_t)g];
        out.reserve(raw[(size_t)g].size());
        bool last_direct = false;
        for (int32_t e : raw[(size_t)g]) {
            if (e == BREAK) {
                last_direct = false;
                continue;
            }
            int64_t start, cnt;
            if (e < 0) {
                start = n_src + (int64_t)slot_of[-1 - e] * m;
                cnt = m;
                far_pairs += cnt;
            } else {
                start = t->nodes[e].begin;
                cnt = t->nodes[e].end - t->nodes[e].begin;
                near_pairs += cnt;
            }
            // contiguous particle ranges merge, proxies do not (tree.cu traverse_kernel)
            if (e >= 0 && last_direct && out.back().first + out.back().second == start &&
                out.back().second + cnt < (1LL << 30))
                out.back().second += (int32_t)cnt;
            else
                out.emplace_back(start, (int32_t)cnt);
            last_direct = e >= 0;
        }
        std::vector<int32_t>().swap(raw[(size_t)g]);
    }
    t->seg_off.assign((size_t)n_groups + 1, 0);
    for (int64_t g = 0; g < n_groups; ++g)
        t->seg_off[g + 1] = t->seg_off[g] + (int64_t)segs[(size_t)g].size();
    const int64_t n_seg = t->seg_off[n_groups];
    t->seg_start.resize((size_t)n_seg);
    t->seg_count.resize((size_t)n_seg);
    for (int64_t g = 0; g < n_groups; ++g) {
        int64_t o = t->seg_off[g];
        for (const auto& sc : segs[(size_t)g]) {
            t->seg_start[o] = sc.first;
            t->seg_count[o] = sc.second;
            ++o;
        }
    }
    t->near_pairs = near_pairs;
    t->far_pairs = far_pairs;
    counts[0] = n_seg;
    counts[1] = n_slots;
    counts[2] = (int64_t)t->unit_slot.size();
    counts[3] = near_pairs;
    counts[4] = far_pairs;
    return SPK_OK;
}

/* Node id behind every proxy slot (for tests / diagnostics). */
void spk_tree_host_slot_nodes(const void* h, int32_t* slot_node) {
    const HostTree* t = static_cast<const HostTree*>(h);
    if (!t->slot_node.empty())
        std::memcpy(slot_node, t->slot_node.data(), t->slot_node.size() * sizeof(int32_t));
}

/* Copy the plan out (sizes from spk_tree_host_plan's counts). */
void spk_tree_host_export_plan(const void* h, int64_t* seg_off, int64_t* seg_start,
                               int32_t* seg_count, float* slot_box, int32_t* unit_slot,
                               int64_t* unit_begin, int64_t* unit_end,
                               int64_t* slot_unit_off) {
    const HostTree* t = static_cast<const HostTree*>(h);
    auto cp = [](auto* dst, const auto& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(seg_off, t->seg_off);
    cp(seg_start, t->seg_start);
    cp(seg_count, t->seg_count);
    cp(slot_box, t->slot_box);
    cp(unit_slot, t->unit_slot);
    cp(unit_begin, t->unit_begin);
    cp(unit_end, t->unit_end);
    cp(slot_unit_off, t->slot_unit_off);
}

}  // extern "C"
