// TEST INFRASTRUCTURE — oracle only. Never linked into the product.
//
// Restatement of the boost::dynamic_bitset subset used by the reference's
// DagTask (dag.hpp:89-90; dag.cpp:112-135, 179-208): construction with a
// size, |, |=, set, test, find_first, find_next, npos. Boost itself is not
// installed in this image; version used by the reference is unpinned.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

namespace boost {

template <typename Block = unsigned long, typename Allocator = std::allocator<Block>>
class dynamic_bitset {
  public:
    using size_type = std::size_t;
    static constexpr size_type npos = static_cast<size_type>(-1);

    dynamic_bitset() = default;
    explicit dynamic_bitset(size_type n) : bits_(n), words_((n + 63) / 64, 0) {}

    size_type size() const { return bits_; }
    dynamic_bitset& set(size_type i) {
        words_[i >> 6] |= std::uint64_t(1) << (i & 63);
        return *this;
    }
    bool test(size_type i) const { return (words_[i >> 6] >> (i & 63)) & 1; }

    dynamic_bitset& operator|=(const dynamic_bitset& o) {
        for (size_type w = 0; w < words_.size(); ++w) words_[w] |= o.words_[w];
        return *this;
    }
    friend dynamic_bitset operator|(const dynamic_bitset& a, const dynamic_bitset& b) {
        dynamic_bitset r = a;
        r |= b;
        return r;
    }

    size_type find_first() const { return scan(0); }
    size_type find_next(size_type pos) const { return pos + 1 >= bits_ ? npos : scan(pos + 1); }

  private:
    size_type scan(size_type from) const {
        for (size_type w = from >> 6; w < words_.size(); ++w) {
            std::uint64_t word = words_[w];
            if (w == (from >> 6)) word &= ~std::uint64_t(0) << (from & 63);
            if (word) {
                size_type i = (w << 6) + static_cast<size_type>(__builtin_ctzll(word));
                return i < bits_ ? i : npos;
            }
        }
        return npos;
    }

    size_type bits_ = 0;
    std::vector<std::uint64_t> words_;
};

}  // namespace boost
