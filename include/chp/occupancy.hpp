// chp/occupancy.hpp -- drop-in for /root/reference/proj/include/chp/occupancy.hpp:1-230.
// Same API (the paper's bit array M and the w-ary summary tree, section 4);
// independent implementation.  On the device the bit array is produced by
// the compaction kernel K3 (csrc/compact.cu) as 64-bit words in exactly
// the BlockedBitset<uint64_t> layout; assign_words() (an extension, not in
// the reference) installs those words without one insert() per slot.
#pragma once

#include <bit>
#include <concepts>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace chp::occupancy {

template <typename Word>
concept BitWord = std::unsigned_integral<Word> && !std::same_as<Word, bool>;

// Positions of the set bits of x, lowest first.
template <BitWord Word>
std::vector<int> extract_word_positions(Word x) {
    std::vector<int> out;
    out.reserve(static_cast<std::size_t>(std::popcount(x)));
    for (; x; x &= static_cast<Word>(x - 1)) out.push_back(std::countr_zero(x));
    return out;
}

// Index of the highest set bit (x != 0).
template <BitWord Word>
int msb_position(Word x) {
    return static_cast<int>(sizeof(Word) * 8) - 1 - std::countl_zero(x);
}

struct BlockPosition {
    std::uint64_t block;
    std::uint32_t position;

    friend bool operator==(const BlockPosition&, const BlockPosition&) = default;
};

// 1-based slot i -> (word, bit) for power-of-two word width w.
inline BlockPosition bit_index_map(std::uint64_t i, std::uint32_t w) {
    const std::uint64_t z = i - 1;
    return {z / w, static_cast<std::uint32_t>(z % w)};
}

// The paper's sparsity condition p < n (w + 1).
inline bool practical_linearity_check(std::uint64_t n, std::uint64_t p, std::uint32_t w) {
    using u128 = unsigned __int128;
    return static_cast<u128>(p) < static_cast<u128>(n) * (static_cast<u128>(w) + 1);
}

template <BitWord Word>
class BlockedBitset {
  public:
    static constexpr std::uint32_t word_bits = sizeof(Word) * 8;

    explicit BlockedBitset(std::uint64_t p) : p_(p), words_((p + word_bits - 1) / word_bits) {}

    std::uint64_t size() const { return p_; }
    std::uint64_t block_count() const { return words_.size(); }
    const std::vector<Word>& blocks() const { return words_; }

    void insert(std::uint64_t i) {
        guard(i);
        words_[(i - 1) / word_bits] |= static_cast<Word>(Word{1} << ((i - 1) % word_bits));
    }
    bool test(std::uint64_t i) const {
        guard(i);
        return (words_[(i - 1) / word_bits] >> ((i - 1) % word_bits)) & Word{1};
    }

    // Extension: install device-produced words (BlockedBitset layout).
    void assign_words(const Word* w, std::size_t count) {
        if (count != words_.size()) throw std::invalid_argument("BlockedBitset: word count mismatch");
        for (std::size_t k = 0; k < count; ++k) words_[k] = w[k];
    }

    template <typename F>
    void for_each(F&& f) const {
        for (std::uint64_t b = 0; b < words_.size(); ++b)
            for (Word x = words_[b]; x; x &= static_cast<Word>(x - 1))
                f(b * word_bits + static_cast<std::uint64_t>(std::countr_zero(x)) + 1);
    }

    std::vector<std::uint64_t> indices() const {
        std::vector<std::uint64_t> out;
        for_each([&](std::uint64_t i) { out.push_back(i); });
        return out;
    }

  private:
    void guard(std::uint64_t i) const {
        if (i == 0 || i > p_) throw std::out_of_range("BlockedBitset: index out of range");
    }
    std::uint64_t p_;
    std::vector<Word> words_;
};

// Summary tree: level 0 is the bit array, each word of level L+1 has bit j
// set iff word j of its child range on level L is non-zero.  All levels live
// in one vector; offsets_[L] is where level L starts.
template <BitWord Word>
class WAryOccupancyTree {
  public:
    static constexpr std::uint32_t word_bits = sizeof(Word) * 8;

    explicit WAryOccupancyTree(std::uint64_t p) : p_(p) {
        std::uint64_t n = (p + word_bits - 1) / word_bits;
        std::uint64_t at = 0;
        for (;;) {
            offsets_.push_back(at);
            counts_.push_back(n);
            at += n;
            if (n <= 1) break;
            n = (n + word_bits - 1) / word_bits;
        }
        words_.assign(at, Word{0});
    }

    std::uint64_t size() const { return p_; }
    std::uint64_t height() const { return counts_.size() - 1; }
    std::uint64_t total_words() const { return words_.size(); }
    std::uint64_t leaf_words() const { return counts_.front(); }

    void insert(std::uint64_t i) {
        if (i == 0 || i > p_) throw std::out_of_range("WAryOccupancyTree: index out of range");
        std::uint64_t bit = i - 1;
        for (std::size_t L = 0; L < counts_.size(); ++L) {
            words_[offsets_[L] + bit / word_bits] |= static_cast<Word>(Word{1} << (bit % word_bits));
            bit /= word_bits;
        }
    }
    bool test(std::uint64_t i) const {
        if (i == 0 || i > p_) throw std::out_of_range("WAryOccupancyTree: index out of range");
        return (words_[(i - 1) / word_bits] >> ((i - 1) % word_bits)) & Word{1};
    }

    // Depth-first over non-zero children only, with an explicit stack.
    template <typename F>
    void for_each(F&& f) const {
        struct Frame {
            std::size_t level;
            std::uint64_t word;
            Word rest;
        };
        std::vector<Frame> st;
        const std::size_t top = counts_.size() - 1;
        st.push_back({top, 0, words_[offsets_[top]]});
        while (!st.empty()) {
            Frame& fr = st.back();
            if (!fr.rest) {
                st.pop_back();
                continue;
            }
            const std::uint64_t child = fr.word * word_bits + static_cast<std::uint64_t>(std::countr_zero(fr.rest));
            fr.rest &= static_cast<Word>(fr.rest - 1);
            if (fr.level == 0) {
                f(child + 1);
            } else {
                const std::size_t L = fr.level - 1;
                st.push_back({L, child, words_[offsets_[L] + child]});
            }
        }
    }

    std::vector<std::uint64_t> indices() const {
        std::vector<std::uint64_t> out;
        for_each([&](std::uint64_t i) { out.push_back(i); });
        return out;
    }

  private:
    std::uint64_t p_;
    std::vector<std::uint64_t> offsets_, counts_;
    std::vector<Word> words_;
};

enum class Kind { array, tree };

// Either structure over 64-bit words, chosen at construction.
class Index {
  public:
    Index(std::uint64_t p, Kind kind)
        : kind_(kind),
          array_(kind == Kind::array ? p : 0),
          tree_(kind == Kind::tree ? p : 0) {}

    Kind kind() const { return kind_; }

    void insert(std::uint64_t i) {
        if (kind_ == Kind::array)
            array_.insert(i);
        else
            tree_.insert(i);
    }
    bool test(std::uint64_t i) const { return kind_ == Kind::array ? array_.test(i) : tree_.test(i); }

    template <typename F>
    void for_each(F&& f) const {
        if (kind_ == Kind::array)
            array_.for_each(f);
        else
            tree_.for_each(f);
    }

    std::vector<std::uint64_t> indices() const {
        return kind_ == Kind::array ? array_.indices() : tree_.indices();
    }

    // Extension: install BlockedBitset<uint64_t> words from the device.
    void assign_words(const std::uint64_t* w, std::size_t count) {
        if (kind_ == Kind::array) {
            array_.assign_words(w, count);
            return;
        }
        for (std::size_t b = 0; b < count; ++b)
            for (std::uint64_t x = w[b]; x; x &= x - 1)
                tree_.insert(b * 64 + static_cast<std::uint64_t>(std::countr_zero(x)) + 1);
    }

  private:
    Kind kind_;
    BlockedBitset<std::uint64_t> array_;
    WAryOccupancyTree<std::uint64_t> tree_;
};

}  // namespace chp::occupancy
