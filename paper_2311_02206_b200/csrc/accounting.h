// accounting.h — host bookkeeping the drop-in must preserve (SURVEY §8a
// rows a18/a19): the logical-byte memory accountant (budget.hpp:16-112) and
// the Eager Buffer Management policy of the merge buffers
// (merge_buffer.hpp:29-117, paper Alg. 2).  These are restated here (not
// copied) so run_stats — peak_tracked_bytes, peak_temp_bytes,
// charge_events, buffer_allocations — and every budget_error(phase) match
// the reference engine charge for charge.  The EBM capacity also sizes the
// device merge target of each relation (engine.cu).
#pragma once

#include <stdint.h>

#include <map>
#include <string>

#include "ctx.h"

namespace gd {

class Accountant {
public:
    enum Cat { kContainer = 0, kTemp = 1, kBuffer = 2 };
    static constexpr uint64_t kUnlimited = UINT64_MAX;

    explicit Accountant(uint64_t budget = kUnlimited) : budget_(budget) {}

    bool can_charge(uint64_t bytes) const {  // budget.hpp:24-27
        if (budget_ == kUnlimited) return true;
        return total() + bytes <= budget_;
    }
    void charge(Cat cat, uint64_t bytes, const char* phase) {  // budget.hpp:29-43
        if (bytes == 0) return;
        if (!can_charge(bytes))
            throw_budget(phase, "need " + std::to_string(bytes) + " more bytes with " +
                                    std::to_string(total()) + " in use of " +
                                    std::to_string(budget_) + " budgeted");
        cur_[cat] += bytes;
        ++events_;
        if (total() > peak_) peak_ = total();
        if (cat == kTemp && cur_[cat] > peak_temp_) peak_temp_ = cur_[cat];
    }
    void release(Cat cat, uint64_t bytes) {  // budget.hpp:45-48
        uint64_t& c = cur_[cat];
        c = bytes > c ? 0 : c - bytes;
    }
    uint64_t current(Cat cat) const { return cur_[cat]; }
    uint64_t total() const { return cur_[0] + cur_[1] + cur_[2]; }
    uint64_t peak() const { return peak_; }
    uint64_t peak_temp() const { return peak_temp_; }
    uint64_t events() const { return events_; }
    uint64_t budget() const { return budget_; }

private:
    uint64_t budget_;
    uint64_t cur_[3] = {0, 0, 0};
    uint64_t peak_ = 0, peak_temp_ = 0, events_ = 0;
};

// RAII charge (tracked_bytes, budget.hpp:71-112).
class Tracked {
public:
    Tracked() = default;
    Tracked(Accountant& a, Accountant::Cat cat, uint64_t bytes, const char* phase) : a_(&a), cat_(cat) {
        a.charge(cat, bytes, phase);
        bytes_ = bytes;
    }
    Tracked(Tracked&& o) noexcept : a_(o.a_), cat_(o.cat_), bytes_(o.bytes_) {
        o.a_ = nullptr;
        o.bytes_ = 0;
    }
    Tracked& operator=(Tracked&& o) noexcept {
        if (this != &o) {
            reset();
            a_ = o.a_; cat_ = o.cat_; bytes_ = o.bytes_;
            o.a_ = nullptr; o.bytes_ = 0;
        }
        return *this;
    }
    Tracked(const Tracked&) = delete;
    Tracked& operator=(const Tracked&) = delete;
    ~Tracked() { reset(); }
    void reset() {
        if (a_ && bytes_) a_->release(cat_, bytes_);
        a_ = nullptr;
        bytes_ = 0;
    }
    uint64_t bytes() const { return bytes_; }

private:
    Accountant* a_ = nullptr;
    Accountant::Cat cat_ = Accountant::kContainer;
    uint64_t bytes_ = 0;
};

// EBM (merge_buffer.hpp:29-117): one retained buffer per relation.
class BufferManager {
public:
    BufferManager(Accountant& a, bool eager, unsigned alpha) : acct_(&a), eager_(eager), alpha_(alpha) {
        if (alpha_ == 0) throw_config("buffer_manager: alpha must be at least 1");
    }

    // Returns the buffer capacity in rows after the acquire.
    uint64_t acquire(const std::string& rel, uint64_t full_rows, uint64_t delta_rows, uint32_t arity) {
        Buf& b = bufs_[rel];
        if (b.in_use) throw_logic("buffer_manager: buffer already in use");
        const uint64_t need = full_rows + delta_rows;
        if (eager_ && b.arity == arity && b.capacity >= need) {
            b.in_use = true;
            return b.capacity;
        }
        const uint64_t old_bytes = charges_[rel].bytes();
        uint64_t rows = 0;
        if (eager_) {
            for (unsigned k = alpha_; k >= 1; --k) {
                const uint64_t cand = full_rows + delta_rows * k;
                const uint64_t bytes = cand * arity * 8;
                if (acct_->can_charge(bytes > old_bytes ? bytes - old_bytes : 0)) {
                    rows = cand;
                    break;
                }
            }
            if (rows == 0)
                throw_budget("merge", "not enough memory for the merge buffer of '" + rel + "' (full " +
                                          std::to_string(full_rows) + " rows, delta " +
                                          std::to_string(delta_rows) + " rows)");
        } else {
            rows = need;
        }
        charges_[rel].reset();
        charges_[rel] = Tracked(*acct_, Accountant::kBuffer, rows * arity * 8, "merge");
        b.arity = arity;
        b.capacity = rows;
        b.in_use = true;
        ++allocations_;
        return rows;
    }
    void release(const std::string& rel) {
        auto it = bufs_.find(rel);
        if (it == bufs_.end() || !it->second.in_use) throw_logic("buffer_manager: release without acquire");
        it->second.in_use = false;
        if (!eager_) {
            charges_[rel].reset();
            it->second.capacity = 0;
        }
    }
    uint64_t allocations() const { return allocations_; }
    bool eager() const { return eager_; }
    unsigned alpha() const { return alpha_; }

private:
    struct Buf {
        uint32_t arity = 0;
        uint64_t capacity = 0;
        bool in_use = false;
    };
    Accountant* acct_;
    bool eager_;
    unsigned alpha_;
    uint64_t allocations_ = 0;
    std::map<std::string, Buf> bufs_;
    std::map<std::string, Tracked> charges_;
};

}  // namespace gd
