// plan.cpp -- blocking plan, exponents, root owners and packed offsets (row a1).
//
// Rule (readings #5, #12, #13, #17):
//  * side kept iff 1 < dim <= max_precond_dim (bypass huge dims);
//  * both kept -> p = 4 / 4; one kept -> p = 2 on it;
//    a split (a, d) gives the two-sided exponents a/(2d) and (d-a)/(2d) stored
//    reduced as r/p (f4; reading #23);
//  * each axis split into ceil(dim/b) contiguous ranges, last ragged,
//    blocks row-major over the block grid, tensors in caller order;
//  * roots sorted by (cost desc, tensor, block, side) with cost = n^3 * products
//    per Newton iteration, assigned LPT to the least-loaded rank;
//  * packing: rank-major segments of equal size; inside a segment groups of
//    equal (n, p, r) in (n desc, p desc, r desc) order; ld = roundup(n, 4), group stride
//    roundup(n*ld, 64); segment size roundup(max used, 64).
#include <algorithm>
#include <cstring>
#include <tuple>
#include <vector>

#include "internal.h"

namespace shp {

static int64_t roundup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// X*T, the left-to-right binary chain for T^p (bitlen-1 squarings, popcount-1
// multiplications by T) and T^p*M
static int64_t products_per_iteration(int p) {
  int bits = 0, ones = 0;
  for (int q = p; q; q >>= 1) {
    ++bits;
    ones += q & 1;
  }
  return 2 + (bits - 1) + (ones - 1);
}

static int gcd_i(int a, int b) { return b ? gcd_i(b, a % b) : a; }

struct RootRef {
  int64_t cost;
  int32_t tensor, block, side;
  int32_t n, p, r;
};

// Roots sorted by (cost desc, tensor, block, side/mode), assigned LPT to the
// least-loaded rank (lowest rank on ties), then packed per rank: groups of
// equal (n, p, r) in (n desc, p desc, r desc) order, ld = roundup(n, 4), group
// stride roundup(n*ld, 64); segments padded to the largest (roundup 64).
// set(root, owner, absolute offset, ld) records each root's placement.
// Returns the segment size.
// tensor_owner (optional): every root of tensor t goes to tensor_owner[t] instead of the per-root LPT
// (layer-granular distribution, reading #30).
template <class Set>
static int64_t assign_and_pack(std::vector<RootRef>& roots, int world_size, std::vector<shampoo_group_t>& groups,
                               Set set, const std::vector<int>* tensor_owner = nullptr) {
  std::stable_sort(roots.begin(), roots.end(), [](const RootRef& x, const RootRef& y) {
    return std::make_tuple(-x.cost, x.tensor, x.block, x.side) < std::make_tuple(-y.cost, y.tensor, y.block, y.side);
  });
  std::vector<int64_t> load(world_size, 0);
  std::vector<std::vector<int32_t>> owned(world_size);  // sorted positions
  std::vector<int> owner_of(roots.size(), 0);
  for (int32_t pos = 0; pos < (int32_t)roots.size(); ++pos) {
    int r = 0;
    if (tensor_owner) {
      r = (*tensor_owner)[roots[pos].tensor];
    } else {
      for (int q = 1; q < world_size; ++q)
        if (load[q] < load[r]) r = q;
    }
    load[r] += roots[pos].cost;
    owned[r].push_back(pos);
    owner_of[pos] = r;
  }
  std::vector<int64_t> used(world_size, 0), rel_off(roots.size(), 0), ld_of(roots.size(), 0);
  const size_t g0 = groups.size();
  for (int r = 0; r < world_size; ++r) {
    std::vector<int32_t> items = owned[r];
    std::stable_sort(items.begin(), items.end(), [&](int32_t a, int32_t c) {
      const RootRef& x = roots[a];
      const RootRef& y = roots[c];
      return std::make_tuple(-x.n, -x.p, -x.r, a) < std::make_tuple(-y.n, -y.p, -y.r, c);
    });
    int64_t off = 0;
    size_t i = 0;
    while (i < items.size()) {
      const int32_t n = roots[items[i]].n, p = roots[items[i]].p, rr = roots[items[i]].r;
      size_t j = i;
      while (j < items.size() && roots[items[j]].n == n && roots[items[j]].p == p && roots[items[j]].r == rr) ++j;
      const int64_t ld = roundup(n, 4), stride = roundup((int64_t)n * ld, 64);
      shampoo_group_t g;
      g.owner = r;
      g.n = n;
      g.p = p;
      g.r = rr;
      g.reserved = 0;
      g.count = (int32_t)(j - i);
      g.offset = off;  // relative to the segment for now
      g.stride = stride;
      groups.push_back(g);
      for (size_t k = i; k < j; ++k) {
        rel_off[items[k]] = off + (int64_t)(k - i) * stride;
        ld_of[items[k]] = ld;
      }
      off += (int64_t)(j - i) * stride;
      i = j;
    }
    used[r] = off;
  }
  const int64_t seg = roundup(world_size ? *std::max_element(used.begin(), used.end()) : 0, 64);
  for (size_t q = g0; q < groups.size(); ++q) groups[q].offset += (int64_t)groups[q].owner * seg;
  for (size_t pos = 0; pos < roots.size(); ++pos)
    set(roots[pos], owner_of[pos], rel_off[pos] + (int64_t)owner_of[pos] * seg, (int)ld_of[pos]);
  return seg;
}

// Layer-granular owners (reading #30): tensors sorted by (cost desc, index) with cost = sum over their roots of
// n^3 (products per iteration + 12) -- on the Ozaki path a root's time hardly depends on p (measured per 1024^2
// root: p = 4 0.96-1.04 ms, p = 2 1.03-1.10 ms, more iterations and small-batch costs; products alone would say
// 0.75), so a large p-independent term; K >= 12 all give the same order for Transformer-Big -- plus m*n (so
// tensors without a preconditioned side still spread), each assigned to the least-loaded rank (lowest on ties).
static std::vector<int> tensor_owners(const std::vector<RootRef>& roots, const int64_t* shapes, int32_t n_tensors,
                                      int world_size) {
  std::vector<int64_t> cost(n_tensors, 0);
  for (int32_t t = 0; t < n_tensors; ++t) cost[t] = shapes[2 * t] * shapes[2 * t + 1];
  for (const RootRef& r : roots) cost[r.tensor] += (int64_t)r.n * r.n * r.n * (products_per_iteration(r.p) + 12);
  std::vector<int32_t> order(n_tensors);
  for (int32_t t = 0; t < n_tensors; ++t) order[t] = t;
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return std::make_tuple(-cost[a], a) < std::make_tuple(-cost[b], b); });
  std::vector<int64_t> load(world_size, 0);
  std::vector<int> owner(n_tensors, 0);
  for (int32_t t : order) {
    int r = 0;
    for (int q = 1; q < world_size; ++q)
      if (load[q] < load[r]) r = q;
    load[r] += cost[t];
    owner[t] = r;
  }
  return owner;
}

int plan_impl(const int64_t* shapes, int32_t n_tensors, int32_t block_size, int64_t max_precond_dim,
              int32_t world_size, int32_t split_num, int32_t split_den, shampoo_block_t* out_blocks, int32_t capacity, int32_t* n_blocks_out,
              shampoo_group_t* out_groups, int32_t group_capacity, int32_t* n_groups_out, int64_t* stats_elems,
              int64_t* segment_elems, int32_t layer_owners, int32_t* tensor_owner_out) {
  if (!shapes || n_tensors < 0 || block_size < 1 || max_precond_dim < 1 || world_size < 1)
    return set_error(SHAMPOO_ERR_INVALID_ARG, "plan: bad arguments");
  if (split_num < 1 || split_num >= split_den)
    return set_error(SHAMPOO_ERR_INVALID_ARG, "plan: split needs 1 <= split_num < split_den");
  const int gl = gcd_i(split_num, 2 * split_den), gr = gcd_i(split_den - split_num, 2 * split_den);
  const int p2l = 2 * split_den / gl, r2l = split_num / gl;
  const int p2r = 2 * split_den / gr, r2r = (split_den - split_num) / gr;
  if (p2l > 16 || p2r > 16) return set_error(SHAMPOO_ERR_INVALID_ARG, "plan: split needs root orders <= 16");
  std::vector<shampoo_block_t> blocks;
  for (int32_t t = 0; t < n_tensors; ++t) {
    const int64_t m = shapes[2 * t], n = shapes[2 * t + 1];
    if (m < 1 || n < 1) return set_error(SHAMPOO_ERR_INVALID_ARG, "plan: tensor %d has a zero dimension", t);
    const bool left = m > 1 && m <= max_precond_dim;
    const bool right = n > 1 && n <= max_precond_dim;
    const int pl = left ? (right ? p2l : 2) : 0, rl = left ? (right ? r2l : 1) : 0;
    const int pr = right ? (left ? p2r : 2) : 0, rr = right ? (left ? r2r : 1) : 0;
    for (int64_t r0 = 0; r0 < m; r0 += block_size)
      for (int64_t c0 = 0; c0 < n; c0 += block_size) {
        shampoo_block_t b;
        std::memset(&b, 0, sizeof b);
        b.tensor_id = t;
        b.row0 = r0;
        b.col0 = c0;
        b.rows = (int32_t)std::min<int64_t>(block_size, m - r0);
        b.cols = (int32_t)std::min<int64_t>(block_size, n - c0);
        b.p_left = pl;
        b.p_right = pr;
        b.r_left = rl;
        b.r_right = rr;
        b.owner_left = b.owner_right = -1;
        b.left_off = b.right_off = -1;
        b.left_ld = b.right_ld = 0;
        blocks.push_back(b);
      }
  }
  std::vector<RootRef> roots;
  for (int32_t i = 0; i < (int32_t)blocks.size(); ++i) {
    const shampoo_block_t& b = blocks[i];
    if (b.p_left) {
      const int64_t n = b.rows;
      roots.push_back({n * n * n * products_per_iteration(b.p_left), b.tensor_id, i, 0, b.rows, b.p_left, b.r_left});
    }
    if (b.p_right) {
      const int64_t n = b.cols;
      roots.push_back({n * n * n * products_per_iteration(b.p_right), b.tensor_id, i, 1, b.cols, b.p_right, b.r_right});
    }
  }
  std::vector<shampoo_group_t> groups;
  std::vector<int> towner;
  if (layer_owners) towner = tensor_owners(roots, shapes, n_tensors, world_size);
  if (tensor_owner_out && layer_owners)
    for (int32_t t = 0; t < n_tensors; ++t) tensor_owner_out[t] = towner[t];
  const int64_t seg = assign_and_pack(roots, world_size, groups, [&](const RootRef& rr, int owner, int64_t off, int ld) {
    shampoo_block_t& b = blocks[rr.block];
    if (rr.side == 0) {
      b.owner_left = owner;
      b.left_off = off;
      b.left_ld = ld;
    } else {
      b.owner_right = owner;
      b.right_off = off;
      b.right_ld = ld;
    }
  }, layer_owners ? &towner : nullptr);
  if (n_blocks_out) *n_blocks_out = (int32_t)blocks.size();
  if (n_groups_out) *n_groups_out = (int32_t)groups.size();
  if (stats_elems) *stats_elems = seg * world_size;
  if (segment_elems) *segment_elems = seg;
  bool cap_ok = true;
  if (out_blocks) {
    if (capacity < (int32_t)blocks.size()) cap_ok = false;
    else std::memcpy(out_blocks, blocks.data(), blocks.size() * sizeof(shampoo_block_t));
  }
  if (out_groups) {
    if (group_capacity < (int32_t)groups.size()) cap_ok = false;
    else std::memcpy(out_groups, groups.data(), groups.size() * sizeof(shampoo_group_t));
  }
  if (!cap_ok) return set_error(SHAMPOO_ERR_CAPACITY, "plan: output capacity too small (%zu blocks, %zu groups)",
                                blocks.size(), groups.size());
  return SHAMPOO_OK;
}

// ------------------------------------------------------------- f3: tensors
// Rule (oracle/tensor.py; readings #24-#26): mode i kept iff 1 < d_i <=
// max_precond_dim, p = 2 * (#kept) on every kept mode; every mode split into
// ceil(d_i / b) ranges, blocks row-major over the block grid; roots and
// packing exactly as the matrix plan (side = mode).
int tensor_plan_impl(const int64_t* dims, const int32_t* orders, int32_t n_tensors, int32_t block_size,
                     int64_t max_precond_dim, int32_t world_size, shampoo_tblock_t* out_blocks, int32_t capacity,
                     int32_t* n_blocks_out, shampoo_group_t* out_groups, int32_t group_capacity,
                     int32_t* n_groups_out, int64_t* stats_elems, int64_t* segment_elems) {
  constexpr int K = SHAMPOO_MAX_ORDER;
  if (!dims || !orders || n_tensors < 0 || block_size < 1 || max_precond_dim < 1 || world_size < 1)
    return set_error(SHAMPOO_ERR_INVALID_ARG, "tensor plan: bad arguments");
  std::vector<shampoo_tblock_t> blocks;
  for (int32_t t = 0; t < n_tensors; ++t) {
    const int k = orders[t];
    if (k < 1 || k > K) return set_error(SHAMPOO_ERR_INVALID_ARG, "tensor plan: tensor %d has order %d", t, k);
    const int64_t* d = dims + (int64_t)K * t;
    int kept = 0;
    int64_t grid[K], total = 1;
    for (int i = 0; i < k; ++i) {
      if (d[i] < 1) return set_error(SHAMPOO_ERR_INVALID_ARG, "tensor plan: tensor %d has a zero dimension", t);
      kept += (d[i] > 1 && d[i] <= max_precond_dim) ? 1 : 0;
      grid[i] = (d[i] + block_size - 1) / block_size;
      total *= grid[i];
    }
    for (int64_t flat = 0; flat < total; ++flat) {
      shampoo_tblock_t b;
      std::memset(&b, 0, sizeof b);
      b.tensor_id = t;
      b.order = k;
      int64_t rem = flat;
      for (int i = k - 1; i >= 0; --i) {
        const int64_t idx = rem % grid[i];
        rem /= grid[i];
        b.origin[i] = idx * block_size;
        b.extent[i] = (int32_t)std::min<int64_t>(block_size, d[i] - b.origin[i]);
      }
      for (int i = 0; i < K; ++i) {
        if (i >= k) b.extent[i] = 1;
        b.p[i] = (i < k && d[i] > 1 && d[i] <= max_precond_dim) ? 2 * kept : 0;
        b.owner[i] = -1;
        b.off[i] = -1;
        b.ld[i] = 0;
      }
      blocks.push_back(b);
    }
  }
  std::vector<RootRef> roots;
  for (int32_t i = 0; i < (int32_t)blocks.size(); ++i) {
    const shampoo_tblock_t& b = blocks[i];
    for (int m = 0; m < b.order; ++m)
      if (b.p[m]) {
        const int64_t n = b.extent[m];
        roots.push_back({n * n * n * products_per_iteration(b.p[m]), b.tensor_id, i, m, b.extent[m], b.p[m], 1});
      }
  }
  std::vector<shampoo_group_t> groups;
  const int64_t seg = assign_and_pack(roots, world_size, groups, [&](const RootRef& rr, int owner, int64_t off, int ld) {
    shampoo_tblock_t& b = blocks[rr.block];
    b.owner[rr.side] = owner;
    b.off[rr.side] = off;
    b.ld[rr.side] = ld;
  });
  if (n_blocks_out) *n_blocks_out = (int32_t)blocks.size();
  if (n_groups_out) *n_groups_out = (int32_t)groups.size();
  if (stats_elems) *stats_elems = seg * world_size;
  if (segment_elems) *segment_elems = seg;
  bool cap_ok = true;
  if (out_blocks) {
    if (capacity < (int32_t)blocks.size()) cap_ok = false;
    else std::memcpy(out_blocks, blocks.data(), blocks.size() * sizeof(shampoo_tblock_t));
  }
  if (out_groups) {
    if (group_capacity < (int32_t)groups.size()) cap_ok = false;
    else std::memcpy(out_groups, groups.data(), groups.size() * sizeof(shampoo_group_t));
  }
  if (!cap_ok)
    return set_error(SHAMPOO_ERR_CAPACITY, "tensor plan: output capacity too small (%zu blocks, %zu groups)",
                     blocks.size(), groups.size());
  return SHAMPOO_OK;
}

}  // namespace shp
