// Bit-exact O(log n) replacement for the reference's src/learner/replay_mem.cpp; see
// include/tleague/learner/replay_mem.hpp.
#include "tleague/learner/replay_mem.hpp"

#include <stdexcept>
#include <utility>

namespace tleague::learner {

namespace {
std::size_t PowerOfTwoAtLeast(std::size_t n) {
  std::size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}
}  // namespace

ReplayMem::ReplayMem(std::size_t capacity, std::uint32_t max_reuse, std::uint64_t seed)
    : capacity_(capacity), max_reuse_(max_reuse), rng_(seed) {
  // the reference's argument checks (replay_mem.cpp:8-12)
  if (capacity_ == 0) throw std::invalid_argument("replay capacity must be >= 1");
  if (max_reuse_ == 0) throw std::invalid_argument("max_reuse must be >= 1");
  const std::size_t n = PowerOfTwoAtLeast(2 * capacity_);
  slots_.resize(n);
  tree_.assign(n + 1, 0);
  live_flag_.assign(n, 0);
}

void ReplayMem::TreeAdd(std::size_t pos, int delta) {
  for (std::size_t i = pos + 1; i < tree_.size(); i += i & (~i + 1)) tree_[i] += delta;
}

std::size_t ReplayMem::TreeFindNth(std::size_t n) const {
  // descend from the highest power of two: the largest prefix holding <= n live entries
  std::size_t pos = 0;
  for (std::size_t step = slots_.size(); step > 0; step >>= 1) {
    const std::size_t next = pos + step;
    if (next < tree_.size() && std::size_t(tree_[next]) <= n) {
      pos = next;
      n -= std::size_t(tree_[next]);
    }
  }
  return pos;  // 0-based position of the (n+1)-th live entry
}

void ReplayMem::Compact() {
  std::size_t w = 0;
  for (std::size_t r = 0; r < tail_; ++r) {
    if (!live_flag_[r]) continue;
    if (w != r) slots_[w] = std::move(slots_[r]);
    ++w;
  }
  for (std::size_t i = w; i < tail_; ++i) slots_[i] = Entry{};
  std::fill(live_flag_.begin(), live_flag_.end(), std::uint8_t(0));
  std::fill(live_flag_.begin(), live_flag_.begin() + std::ptrdiff_t(w), std::uint8_t(1));
  // rebuild the tree in O(n): prefix counts over the flags
  std::fill(tree_.begin(), tree_.end(), 0);
  for (std::size_t i = 1; i < tree_.size(); ++i) {
    tree_[i] += live_flag_[i - 1];
    const std::size_t parent = i + (i & (~i + 1));
    if (parent < tree_.size()) tree_[parent] += tree_[i];
  }
  tail_ = w;
}

void ReplayMem::EraseAt(std::size_t pos) {
  slots_[pos] = Entry{};
  live_flag_[pos] = 0;
  TreeAdd(pos, -1);
  --live_;
}

void ReplayMem::Push(TrajectorySegment segment) {
  std::lock_guard lock(mu_);
  received_steps_ += segment.valid_steps;
  if (live_ == capacity_) EraseAt(TreeFindNth(0));  // FIFO: the oldest live entry
  if (tail_ == slots_.size()) Compact();              // >= capacity holes to reclaim
  slots_[tail_] = Entry{std::move(segment), 0};
  live_flag_[tail_] = 1;
  TreeAdd(tail_, +1);
  ++tail_;
  ++live_;
  cv_.notify_all();
}

std::vector<TrajectorySegment> ReplayMem::SampleBlocking(std::size_t n) {
  if (n == 0) throw std::invalid_argument("sample size must be >= 1");
  std::unique_lock lock(mu_);
  cv_.wait(lock, [&] { return shutdown_ || live_ >= n; });
  if (shutdown_) return {};
  std::vector<TrajectorySegment> out;
  out.reserve(n);
  for (std::size_t k = 0; k < n; ++k) {
    // the reference's draw: index into the live entries in insertion order
    std::uniform_int_distribution<std::size_t> pick(0, live_ - 1);
    const std::size_t pos = TreeFindNth(pick(rng_));
    Entry& e = slots_[pos];
    consumed_steps_ += e.segment.valid_steps;
    if (++e.use_count >= max_reuse_) {
      out.push_back(std::move(e.segment));
      EraseAt(pos);
    } else {
      out.push_back(e.segment);
    }
  }
  return out;
}

void ReplayMem::Clear() {
  std::lock_guard lock(mu_);
  for (std::size_t i = 0; i < tail_; ++i) slots_[i] = Entry{};
  std::fill(live_flag_.begin(), live_flag_.end(), std::uint8_t(0));
  std::fill(tree_.begin(), tree_.end(), 0);
  tail_ = 0;
  live_ = 0;
}

void ReplayMem::SetMaxReuse(std::uint32_t max_reuse) {
  if (max_reuse == 0) throw std::invalid_argument("max_reuse must be >= 1");
  std::lock_guard lock(mu_);
  max_reuse_ = max_reuse;
}

void ReplayMem::Shutdown() {
  std::lock_guard lock(mu_);
  shutdown_ = true;
  cv_.notify_all();
}

std::size_t ReplayMem::size() const {
  std::lock_guard lock(mu_);
  return live_;
}

std::uint64_t ReplayMem::received_steps() const {
  std::lock_guard lock(mu_);
  return received_steps_;
}

std::uint64_t ReplayMem::consumed_steps() const {
  std::lock_guard lock(mu_);
  return consumed_steps_;
}

}  // namespace tleague::learner
