// Implementation of the C++ façade (include/pe/pagedevict.hpp) over the
// engine's C-ABI (include/pe.h). Host code here only validates, stages
// the caller's vectors, synchronises and translates status codes; every
// cache mutation, eviction decision, prefill selection and attention runs
// in the engine's sm_100a kernels.
//
// Reference API mapped (proj/core/…):
//   PagePool            page_pool.hpp:19-42, page_pool.cpp:8-61
//   BlockTable          block_table.hpp:21-102, block_table.cpp:10-78
//   importance helpers  importance.hpp:17-48, importance.cpp:11-75
//   policies            policy.hpp:17-122, policy.cpp:18-322
//   attend              attention.hpp:14-38, attention.cpp:15-118
#include "pe/pagedevict.hpp"

#include <algorithm>
#include <array>
#include <charconv>
#include <cmath>
#include <map>
#include <cstdio>
#include <cstring>
#include <limits>
#include <mutex>
#include <numeric>
#include <unordered_map>

namespace pagedevict {

// ---------------------------------------------------------------- status
void throw_status(pe_status st, const std::string& context) {
    std::string what = context + ": " + pe_status_string(st);
    const char* detail = pe_last_error();
    if (detail != nullptr && *detail != '\0') what += " (" + std::string(detail) + ")";
    switch (st) {
    case PE_POOL_EXHAUSTED: throw PoolExhausted(what);
    case PE_INDEX_OUT_OF_RANGE: throw IndexOutOfRange(what);
    case PE_UNKNOWN_POSITION: throw UnknownPosition(what);
    case PE_OVERFLOW: throw Overflow(what);
    case PE_EMPTY_PAGE: throw EmptyPage(what);
    case PE_K_TOO_LARGE: throw KTooLarge(what);
    case PE_NO_ELIGIBLE_PAGE: throw NoEligiblePage(what);
    case PE_BUDGET_INVALID: throw BudgetInvalid(what);
    case PE_EMPTY_CACHE: throw EmptyCache(what);
    case PE_LENGTH_MISMATCH: throw LengthMismatch(what);
    case PE_EMPTY_INPUT: throw EmptyInput(what);
    case PE_IO_ERROR: throw IoError(what);
    default: throw Error(what);
    }
}

namespace {

void check(pe_status st, const char* context) {
    if (st != PE_OK) throw_status(st, context);
}

// one call + its device status (the façade is synchronous, like the reference)
void check_sync(pe_engine* eng, pe_status st, const char* context) {
    check(st, context);
    check(pe_sync(eng), context);
}

std::uint32_t row_align(pe_dtype dtype) { return dtype == PE_DTYPE_BF16 ? 8u : 4u; }

std::uint32_t round_up(std::uint32_t x, std::uint32_t a) { return (x + a - 1) / a * a; }

std::uint16_t to_bf16(float f) {  // round to nearest even
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u) return static_cast<std::uint16_t>(u >> 16);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<std::uint16_t>(u >> 16);
}

float from_bf16(std::uint16_t b) {
    const std::uint32_t u = static_cast<std::uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// Packs rows of `n` tokens into the engine's row format (zero padding to
// `width` floats; bf16 conversion when the pool stores bf16).
void pack_row(const std::vector<float>& src, std::uint32_t width, pe_dtype dtype, std::uint8_t* dst) {
    if (dtype == PE_DTYPE_BF16) {
        auto* d = reinterpret_cast<std::uint16_t*>(dst);
        for (std::uint32_t i = 0; i < width; ++i) d[i] = i < src.size() ? to_bf16(src[i]) : 0;
    } else {
        auto* d = reinterpret_cast<float*>(dst);
        for (std::uint32_t i = 0; i < width; ++i) d[i] = i < src.size() ? src[i] : 0.0f;
    }
}

std::int64_t checked_position(std::uint64_t p) {
    if (p > static_cast<std::uint64_t>(std::numeric_limits<std::int32_t>::max()))
        throw Overflow("token position " + std::to_string(p) + " exceeds the device's int32 positions");
    return static_cast<std::int64_t>(p);
}

}  // namespace

// ---------------------------------------------------------------- Page
const KvVector& Page::at(std::uint32_t slot) const {
    if (!occupied(slot)) throw IndexOutOfRange("slot " + std::to_string(slot) + " is not occupied");
    return *slots_[slot];
}

void Page::write(KvVector kv) {
    if (write_full()) throw Error("page is write-full");
    slots_[cursor_++] = std::move(kv);
    ++fill_;
}

bool Page::evict(std::uint64_t position) {
    for (std::uint32_t s = 0; s < cursor_; ++s) {
        if (slots_[s] && slots_[s]->position == position) {
            slots_[s].reset();
            --fill_;
            return true;
        }
    }
    return false;
}

void Page::reset() {
    for (auto& s : slots_) s.reset();
    cursor_ = fill_ = 0;
}

// ---------------------------------------------------------------- PagePool
struct PagePool::Impl {
    std::size_t capacity = 0;
    std::uint32_t B = 0;
    PoolOptions opt;
    mutable std::recursive_mutex mu;
    pe_engine* eng = nullptr;
    std::uint32_t width = 0;                  // engine row width (floats), 0 until created
    std::uint32_t max_pages = 0;
    std::vector<std::int32_t> free_slots;     // table slots, LIFO
    std::vector<const BlockTable*> owner;     // slot -> live table
    std::vector<Page> snaps;                  // [capacity] host snapshots
    std::vector<std::uint32_t> slot_width;    // [capacity*B] original token width per slot
    std::size_t zero_capacity_allocated = 0;  // capacity == 0 pools never touch the device

    ~Impl() {
        if (eng) pe_engine_destroy(eng);
    }

    // Creates the engine on first use; `want` = width of the token about to
    // be stored (0: none yet).
    pe_engine* engine(std::uint32_t want) {
        if (eng) {
            if (want > width)
                throw LengthMismatch("token width " + std::to_string(want) + " exceeds the pool's row width " +
                                     std::to_string(width));
            return eng;
        }
        std::uint32_t w = opt.row_width ? opt.row_width : (want ? want : 64u);
        if (want > w) throw LengthMismatch("token wider than PoolOptions::row_width");
        w = round_up(w, row_align(opt.dtype));
        const std::uint32_t n_tables = std::max<std::uint32_t>(opt.max_tables, 1);
        std::uint64_t mp = opt.max_pages_per_table ? opt.max_pages_per_table : capacity;
        mp = std::min<std::uint64_t>(mp, std::max<std::uint64_t>(1, (std::uint64_t(64) << 20) / n_tables));
        mp = std::max<std::uint64_t>(mp, 1);
        if (capacity > static_cast<std::size_t>(std::numeric_limits<std::int32_t>::max()))
            throw Overflow("pool capacity exceeds the device's int32 page ids");
        pe_config c{};
        c.n_seqs = static_cast<std::int32_t>(n_tables);
        c.n_layers = 1;
        c.n_kv_heads = 1;
        c.head_dim = static_cast<std::int32_t>(w);
        c.granularity = PE_GRANULARITY_PER_KV_HEAD;
        c.page_size = static_cast<std::int32_t>(B);
        c.cache_budget = static_cast<std::int32_t>(B);  // decisions take the policy's C per call
        c.dtype = opt.dtype;
        c.policy = PE_POLICY_FULL_CACHE;
        c.capacity = static_cast<std::int32_t>(capacity);
        c.max_pages_per_table = static_cast<std::int32_t>(mp);
        c.device = opt.device;
        pe_engine* e = nullptr;
        check(pe_engine_create(&c, &e), "PagePool");
        eng = e;
        width = w;
        max_pages = static_cast<std::uint32_t>(mp);
        return eng;
    }

    std::int32_t take_slot(const BlockTable* t) {
        std::lock_guard lock(mu);
        if (free_slots.empty())
            throw Error("PagePool: more than PoolOptions::max_tables (" + std::to_string(opt.max_tables) +
                        ") live BlockTables");
        const std::int32_t s = free_slots.back();
        free_slots.pop_back();
        owner[s] = t;
        return s;
    }

    void give_slot(std::int32_t s) {
        std::lock_guard lock(mu);
        owner[s] = nullptr;
        free_slots.push_back(s);
    }

    std::uint64_t holes_of(std::int32_t id) const {
        std::uint64_t h = 0;
        if (eng != nullptr) check(pe_read_page_holes(eng, id, 1, &h), "page holes");
        return h;
    }

    // Refreshes snapshot `id` from the device; `cursor` = slots written.
    Page& snapshot(std::uint32_t id, std::uint32_t cursor) {
        Page& pg = snaps[id];
        pg.id_ = id;
        pg.slots_.assign(B, std::nullopt);
        pg.cursor_ = pg.fill_ = 0;
        if (cursor == 0 || eng == nullptr) return pg;
        pe_info info{};
        check(pe_get_info(eng, &info), "page");
        const std::size_t elt = opt.dtype == PE_DTYPE_BF16 ? 2 : 4;
        std::vector<std::uint8_t> bytes(static_cast<std::size_t>(2) * B * info.row_pitch_bytes);
        std::vector<std::int32_t> pos(B);
        std::uint64_t holes = 0;
        check(pe_read_pages(eng, static_cast<std::int32_t>(id), 1, bytes.data()), "page");
        check(pe_read_positions(eng, static_cast<std::int32_t>(id), 1, pos.data(), nullptr, nullptr), "page");
        check(pe_read_page_holes(eng, static_cast<std::int32_t>(id), 1, &holes), "page");
        std::uint32_t fill = 0;
        for (std::uint32_t s = 0; s < cursor; ++s) {
            if (s < 64 && ((holes >> s) & 1u)) continue;  // evicted slot
            ++fill;
            const std::uint32_t n = std::min(slot_width[static_cast<std::size_t>(id) * B + s], width);
            KvVector kv;
            kv.key.resize(n);
            kv.value.resize(n);
            const std::uint8_t* kr = bytes.data() + static_cast<std::size_t>(s) * info.row_pitch_bytes;
            const std::uint8_t* vr = bytes.data() + static_cast<std::size_t>(B + s) * info.row_pitch_bytes;
            for (std::uint32_t i = 0; i < n; ++i) {
                if (elt == 2) {
                    kv.key[i] = from_bf16(reinterpret_cast<const std::uint16_t*>(kr)[i]);
                    kv.value[i] = from_bf16(reinterpret_cast<const std::uint16_t*>(vr)[i]);
                } else {
                    kv.key[i] = reinterpret_cast<const float*>(kr)[i];
                    kv.value[i] = reinterpret_cast<const float*>(vr)[i];
                }
            }
            kv.position = static_cast<std::uint64_t>(pos[s]);
            kv.key_norm = l2_norm(kv.key);
            kv.value_norm = l2_norm(kv.value);
            pg.slots_[s] = std::move(kv);
        }
        pg.cursor_ = cursor;
        pg.fill_ = fill;
        return pg;
    }
};

PagePool::PagePool(std::size_t capacity, std::uint32_t page_size, PoolOptions options)
    : impl_(std::make_unique<Impl>()) {
    if (page_size == 0) throw Error("page size must be positive");
    impl_->capacity = capacity;
    impl_->B = page_size;
    impl_->opt = options;
    const std::uint32_t n_tables = std::max<std::uint32_t>(options.max_tables, 1);
    impl_->owner.assign(n_tables, nullptr);
    for (std::uint32_t s = n_tables; s > 0; --s) impl_->free_slots.push_back(static_cast<std::int32_t>(s - 1));
    impl_->snaps.resize(capacity);
    impl_->slot_width.assign(capacity * page_size, 0);
}

PagePool::~PagePool() = default;

PageId PagePool::allocate() {
    std::lock_guard lock(impl_->mu);
    if (impl_->capacity == 0) throw PoolExhausted();
    std::int32_t id = -1;
    check(pe_pool_allocate(impl_->engine(0), &id), "PagePool::allocate");
    impl_->snapshot(static_cast<std::uint32_t>(id), 0);
    return static_cast<PageId>(id);
}

void PagePool::release(PageId id) {
    std::lock_guard lock(impl_->mu);
    if (id >= impl_->capacity) throw IndexOutOfRange("page id " + std::to_string(id) + " out of range");
    check(pe_pool_release(impl_->engine(0), static_cast<std::int32_t>(id)), "PagePool::release");
}

Page& PagePool::page(PageId id) {
    std::lock_guard lock(impl_->mu);
    if (id >= impl_->capacity) throw IndexOutOfRange("page id " + std::to_string(id) + " out of range");
    // owner lookup: the page's cursor is the owning table's newest fill if it
    // is that table's newest page, B if it is any other mapped page, else 0
    for (const BlockTable* t : impl_->owner) {
        if (t == nullptr) continue;
        const auto& v = t->view();
        for (std::size_t j = 0; j < v.pages.size(); ++j) {
            if (static_cast<PageId>(v.pages[j]) == id) {
                const bool newest = j + 1 == v.pages.size();
                return impl_->snapshot(id, newest ? static_cast<std::uint32_t>(v.newest_fill) : impl_->B);
            }
        }
    }
    return impl_->snapshot(id, 0);
}

const Page& PagePool::page(PageId id) const { return const_cast<PagePool*>(this)->page(id); }

std::uint32_t PagePool::page_size() const { return impl_->B; }

std::size_t PagePool::capacity() const { return impl_->capacity; }

std::size_t PagePool::free_count() const {
    std::lock_guard lock(impl_->mu);
    if (impl_->eng == nullptr) return impl_->capacity;
    std::int32_t n = 0;
    check(pe_read_free_list(impl_->eng, nullptr, &n), "PagePool::free_count");
    return static_cast<std::size_t>(n);
}

std::size_t PagePool::allocated() const { return capacity() - free_count(); }

pe_engine* PagePool::engine() const {
    std::lock_guard lock(impl_->mu);
    return impl_->engine(0);
}

std::uint32_t PagePool::row_width() const { return impl_->width; }

std::uint64_t memory_bytes(std::uint64_t seq_len, std::uint64_t layer_count, std::uint64_t head_count,
                           std::uint64_t head_dim, std::uint64_t bytes_per_scalar) {
    // page_pool.cpp:50-61: 2 * S * L * H * d * bytes, Overflow past 64 bits
    std::uint64_t total = 2;
    for (const std::uint64_t f : {seq_len, layer_count, head_count, head_dim, bytes_per_scalar}) {
        if (f != 0 && total > std::numeric_limits<std::uint64_t>::max() / f)
            throw Overflow("KV cache byte count exceeds 64 bits");
        total *= f;
    }
    return total;
}

// ---------------------------------------------------------------- BlockTable
BlockTable::BlockTable(PagePool& pool) : pool_(&pool) { slot_ = pool.impl().take_slot(this); }

BlockTable::~BlockTable() {
    try {
        clear();
    } catch (...) {
    }
    release_slot();
}

void BlockTable::release_slot() noexcept {
    if (pool_ != nullptr && slot_ >= 0) pool_->impl().give_slot(slot_);
    slot_ = -1;
}

BlockTable::BlockTable(BlockTable&& other) noexcept : pool_(other.pool_), slot_(other.slot_) {
    other.slot_ = -1;
    other.view_ = View{};
    if (pool_ && slot_ >= 0) {
        std::lock_guard lock(pool_->impl().mu);
        pool_->impl().owner[slot_] = this;
    }
}

BlockTable& BlockTable::operator=(BlockTable&& other) noexcept {
    if (this != &other) {
        try {
            clear();
        } catch (...) {
        }
        release_slot();
        pool_ = other.pool_;
        slot_ = other.slot_;
        view_ = View{};
        other.slot_ = -1;
        other.view_ = View{};
        if (pool_ && slot_ >= 0) {
            std::lock_guard lock(pool_->impl().mu);
            pool_->impl().owner[slot_] = this;
        }
    }
    return *this;
}

const BlockTable::View& BlockTable::view() const {
    if (view_.valid) return view_;
    auto& I = pool_->impl();
    std::lock_guard lock(I.mu);
    view_.pages.clear();
    view_.newest_fill = view_.retained = 0;
    if (slot_ >= 0 && I.eng != nullptr) {
        std::int32_t np = 0;
        view_.pages.resize(I.max_pages);
        check(pe_read_table(I.eng, slot_, view_.pages.data(), &np, &view_.newest_fill, &view_.retained),
              "BlockTable");
        view_.pages.resize(static_cast<std::size_t>(np));
    }
    view_.valid = true;
    return view_;
}

AppendOutcome BlockTable::append_token(KvVector kv) {
    if (slot_ < 0) throw Error("BlockTable was moved from");
    if (kv.key.empty() || kv.key.size() != kv.value.size())
        throw LengthMismatch("key and value must have identical nonzero length");
    auto& I = pool_->impl();
    std::lock_guard lock(I.mu);
    if (I.capacity == 0) throw PoolExhausted();
    const std::uint32_t n = static_cast<std::uint32_t>(kv.key.size());
    pe_engine* eng = I.engine(n);
    const std::size_t before = view().pages.size();
    const std::size_t elt = I.opt.dtype == PE_DTYPE_BF16 ? 2 : 4;
    std::vector<std::uint8_t> k(I.width * elt), v(I.width * elt);
    pack_row(kv.key, I.width, I.opt.dtype, k.data());
    pack_row(kv.value, I.width, I.opt.dtype, v.data());
    const std::int64_t pos = checked_position(kv.position);
    invalidate();
    const pe_status st = pe_table_append(eng, 1, &slot_, k.data(), v.data(), &pos, nullptr);
    check(st, "BlockTable::append_token");
    const pe_status dev = pe_sync(eng);
    if (dev == PE_INVALID_STATE) {
        // a table holding the whole pool can only have run out of pages
        if (I.max_pages >= I.capacity) throw PoolExhausted("BlockTable::append_token: page pool exhausted");
        throw Error("BlockTable::append_token: table holds PoolOptions::max_pages_per_table pages");
    }
    if (dev != PE_OK) throw_status(dev, "BlockTable::append_token");
    const View& after = view();
    if (!after.pages.empty() && after.newest_fill > 0) {
        const std::size_t idx = static_cast<std::size_t>(after.pages.back()) * I.B + (after.newest_fill - 1);
        I.slot_width[idx] = n;
    }
    return AppendOutcome{after.pages.size() > before};
}

void BlockTable::free_page(std::size_t logical_index) {
    if (slot_ < 0) throw Error("BlockTable was moved from");
    auto& I = pool_->impl();
    std::lock_guard lock(I.mu);
    const std::size_t n = view().pages.size();
    if (logical_index >= n)
        throw IndexOutOfRange("logical page index " + std::to_string(logical_index) + " out of range, table has " +
                              std::to_string(n) + " pages");
    invalidate();
    check_sync(I.eng, pe_table_free_page(I.eng, slot_, static_cast<std::int32_t>(logical_index), nullptr),
               "BlockTable::free_page");
}

void BlockTable::evict_slot(std::uint64_t position) {
    if (slot_ < 0) throw Error("BlockTable was moved from");
    auto& I = pool_->impl();
    std::lock_guard lock(I.mu);
    if (I.eng == nullptr || position > static_cast<std::uint64_t>(std::numeric_limits<std::int32_t>::max()))
        throw UnknownPosition("no retained token at position " + std::to_string(position));
    invalidate();
    const pe_status st = pe_table_evict_token(I.eng, slot_, PE_TOKEN_AT_POSITION, static_cast<std::int64_t>(position),
                                              -1, -1, nullptr, nullptr);
    check(st, "BlockTable::evict_slot");
    const pe_status dev = pe_sync(I.eng);
    if (dev == PE_UNKNOWN_POSITION)
        throw UnknownPosition("no retained token at position " + std::to_string(position));
    if (dev != PE_OK) throw_status(dev, "BlockTable::evict_slot");
}

std::size_t BlockTable::page_count() const { return view().pages.size(); }

std::size_t BlockTable::retained_len() const { return static_cast<std::size_t>(view().retained); }

const Page& BlockTable::page_at(std::size_t logical_index) const {
    const View& v = view();
    if (logical_index >= v.pages.size())
        throw IndexOutOfRange("logical page index " + std::to_string(logical_index) + " out of range");
    auto& I = pool_->impl();
    std::lock_guard lock(I.mu);
    const bool newest = logical_index + 1 == v.pages.size();
    return I.snapshot(static_cast<std::uint32_t>(v.pages[logical_index]),
                      newest ? static_cast<std::uint32_t>(v.newest_fill) : I.B);
}

PageId BlockTable::physical_id_at(std::size_t logical_index) const {
    const View& v = view();
    if (logical_index >= v.pages.size())
        throw IndexOutOfRange("logical page index " + std::to_string(logical_index) + " out of range");
    return static_cast<PageId>(v.pages[logical_index]);
}

double BlockTable::fragmentation_ratio() const {
    const View& v = view();
    if (v.pages.empty()) return 0.0;
    const double slots = static_cast<double>(v.pages.size()) * pool_->page_size();
    return 1.0 - static_cast<double>(v.retained) / slots;
}

double BlockTable::fragmentation_ratio_excluding_newest() const {
    const View& v = view();
    if (v.pages.size() <= 1) return 0.0;
    auto& I = pool_->impl();
    std::lock_guard lock(I.mu);
    const std::uint64_t h = I.holes_of(v.pages.back());
    std::int32_t newest_fill = 0;
    for (std::int32_t k = 0; k < v.newest_fill; ++k) newest_fill += (k >= 64 || !((h >> k) & 1u));
    const double slots = static_cast<double>(v.pages.size() - 1) * pool_->page_size();
    return 1.0 - static_cast<double>(v.retained - newest_fill) / slots;
}

std::vector<std::uint64_t> BlockTable::retained_positions() const {
    const View& v = view();
    std::vector<std::uint64_t> out;
    out.reserve(static_cast<std::size_t>(v.retained));
    if (v.pages.empty()) return out;
    auto& I = pool_->impl();
    std::lock_guard lock(I.mu);
    std::vector<std::int32_t> pos(I.B);
    for (std::size_t j = 0; j < v.pages.size(); ++j) {
        check(pe_read_positions(I.eng, v.pages[j], 1, pos.data(), nullptr, nullptr), "retained_positions");
        const std::uint64_t h = I.holes_of(v.pages[j]);
        const std::uint32_t cur = j + 1 == v.pages.size() ? static_cast<std::uint32_t>(v.newest_fill) : I.B;
        for (std::uint32_t s = 0; s < cur; ++s)
            if (s >= 64 || !((h >> s) & 1u)) out.push_back(static_cast<std::uint64_t>(pos[s]));
    }
    return out;
}

void BlockTable::clear() {
    if (slot_ < 0 || pool_ == nullptr) return;
    auto& I = pool_->impl();
    std::lock_guard lock(I.mu);
    if (I.eng == nullptr) return;
    invalidate();
    check_sync(I.eng, pe_table_clear(I.eng, slot_, nullptr), "BlockTable::clear");
}

// ---------------------------------------------------------------- importance
double token_importance(const KvVector& kv) { return kv.value_norm / std::max(kv.key_norm, kNormEpsilon); }

TokenScore token_score(const KvVector& kv) { return TokenScore{kv.position, token_importance(kv)}; }

PageScore page_score(const Page& page, std::size_t logical_index) {
    if (page.fill() == 0) throw EmptyPage();
    double sum = 0.0;
    for (std::uint32_t s = 0; s < page.write_cursor(); ++s)
        if (page.occupied(s)) sum += token_importance(page.at(s));
    return PageScore{logical_index, sum / page.fill(), page.fill()};
}

std::vector<PageScore> score_pages(const BlockTable& table) {
    std::vector<PageScore> out;
    const std::size_t n = table.page_count();
    out.reserve(n);
    for (std::size_t j = 0; j < n; ++j) out.push_back(page_score(table.page_at(j), j));
    return out;
}

std::vector<std::uint64_t> rank_tokens(std::span<const TokenScore> scores, std::size_t k) {
    if (k > scores.size())
        throw KTooLarge("k = " + std::to_string(k) + " exceeds " + std::to_string(scores.size()) + " scored tokens");
    std::vector<TokenScore> v(scores.begin(), scores.end());
    const auto lower = [](const TokenScore& a, const TokenScore& b) {
        return a.score < b.score || (a.score == b.score && a.position < b.position);
    };
    std::nth_element(v.begin(), v.begin() + static_cast<std::ptrdiff_t>(k), v.end(), lower);
    std::vector<std::uint64_t> picked;
    picked.reserve(k);
    for (std::size_t i = 0; i < k; ++i) picked.push_back(v[i].position);
    std::sort(picked.begin(), picked.end());
    return picked;
}

std::size_t rank_pages(std::span<const PageScore> scores) {
    if (scores.empty()) throw NoEligiblePage();
    std::size_t best = 0;
    for (std::size_t i = 1; i < scores.size(); ++i) {
        const bool lower = scores[i].score < scores[best].score ||
                           (scores[i].score == scores[best].score &&
                            scores[i].logical_index < scores[best].logical_index);
        if (lower) best = i;
    }
    return scores[best].logical_index;
}

// ---------------------------------------------------------------- policy
std::string_view to_string(PolicyKind kind) {
    switch (kind) {
    case PolicyKind::PagedEviction: return "paged-eviction";
    case PolicyKind::StreamingLlm: return "streaming-llm";
    case PolicyKind::InvKeyL2: return "inv-key-l2";
    case PolicyKind::KeyDiff: return "key-diff";
    case PolicyKind::FullCache: return "full";
    }
    return "unknown";
}

std::optional<PolicyKind> parse_policy_kind(std::string_view name) {
    for (const PolicyKind k : {PolicyKind::PagedEviction, PolicyKind::StreamingLlm, PolicyKind::InvKeyL2,
                               PolicyKind::KeyDiff, PolicyKind::FullCache})
        if (to_string(k) == name) return k;
    return std::nullopt;
}

void PolicyConfig::validate() const {
    if (page_size == 0) throw BudgetInvalid("page size must be positive");
    if (cache_budget < page_size)
        throw BudgetInvalid("budget must be at least one page (" + std::to_string(page_size) + " tokens)");
    if (cache_budget % page_size != 0) throw BudgetInvalid("budget must be a multiple of page size");
    if (kind == PolicyKind::StreamingLlm && sink_count >= cache_budget)
        throw BudgetInvalid("sink count must be smaller than the budget");
}

PrefillResult EvictionPolicy::prefill_compress(std::vector<KvVector> tokens) const {
    config_.validate();
    if (tokens.empty()) throw Error("prefill requires at least one token");
    if (tokens.size() <= config_.cache_budget) return PrefillResult{std::move(tokens), EvictionDecision::none(0)};
    return compress(std::move(tokens));
}

EvictionDecision EvictionPolicy::decode_step(BlockTable& table, KvVector kv, std::int64_t step) {
    const std::uint64_t newest = kv.position;
    table.append_token(std::move(kv));
    return evict(table, newest, step);
}

namespace {

// Per-process cache of single-table engines that run the prefill scoring and
// selection kernels (K1) for prefill_compress, keyed by row geometry and C.
struct SelectorKey {
    int device;
    std::uint32_t width, B;
    std::size_t C;
    bool operator==(const SelectorKey& o) const {
        return device == o.device && width == o.width && B == o.B && C == o.C;
    }
};
struct SelectorKeyHash {
    std::size_t operator()(const SelectorKey& k) const {
        return std::hash<std::uint64_t>()((std::uint64_t(k.width) << 40) ^ (std::uint64_t(k.B) << 20) ^ k.C ^
                                          (std::uint64_t(k.device) << 60));
    }
};
struct Selectors {
    std::mutex mu;
    std::unordered_map<SelectorKey, pe_engine*, SelectorKeyHash> engines;
};
// intentionally leaked: engines must not be destroyed after the CUDA runtime
// has shut down at process exit
Selectors& selectors() {
    static Selectors* s = new Selectors();
    return *s;
}

}  // namespace

// PagedEviction prefill (policy.cpp:90-101,139-141) on the device: the K1
// kernels score every token (S = ||V|| / max(||K||, eps)), select the
// E = L - C lowest (S, position) and pack the survivors; their positions,
// read back from the packed pages, are the retained set.
std::vector<std::size_t> EvictionPolicy::device_select_survivors(const std::vector<KvVector>& tokens,
                                                                 const PolicyConfig& config) {
    const std::size_t L = tokens.size();
    if (L > static_cast<std::size_t>(std::numeric_limits<std::int32_t>::max()))
        throw Overflow("prefill length exceeds int32");
    std::uint32_t wmax = 0;
    for (const auto& kv : tokens) {
        if (kv.key.empty() || kv.key.size() != kv.value.size())
            throw LengthMismatch("key and value must have identical nonzero length");
        wmax = std::max<std::uint32_t>(wmax, static_cast<std::uint32_t>(kv.key.size()));
    }
    const std::uint32_t W = round_up(wmax, 4);
    // rank order = position order: visit tokens by ascending position (stable)
    std::vector<std::size_t> order(L);
    std::iota(order.begin(), order.end(), std::size_t{0});
    std::stable_sort(order.begin(), order.end(),
                     [&](std::size_t a, std::size_t b) { return tokens[a].position < tokens[b].position; });
    std::vector<float> K(L * W, 0.0f), V(L * W, 0.0f);
    for (std::size_t r = 0; r < L; ++r) {
        const KvVector& kv = tokens[order[r]];
        std::copy(kv.key.begin(), kv.key.end(), K.begin() + static_cast<std::ptrdiff_t>(r * W));
        std::copy(kv.value.begin(), kv.value.end(), V.begin() + static_cast<std::ptrdiff_t>(r * W));
    }
    const std::size_t C = config.cache_budget;
    const std::uint32_t B = config.page_size;
    // the calling thread's current device (one host thread per GPU)
    std::int32_t device = 0;
    check(pe_current_device(&device), "prefill_compress");
    auto& sel = selectors();
    std::lock_guard lock(sel.mu);
    const SelectorKey key{device, W, B, C};
    pe_engine*& eng = sel.engines[key];
    if (eng == nullptr) {
        pe_config c{};
        c.n_seqs = 1;
        c.n_layers = 1;
        c.n_kv_heads = 1;
        c.head_dim = static_cast<std::int32_t>(W);
        c.granularity = PE_GRANULARITY_PER_KV_HEAD;
        c.page_size = static_cast<std::int32_t>(B);
        c.cache_budget = static_cast<std::int32_t>(C);
        c.dtype = PE_DTYPE_F32;
        c.policy = PE_POLICY_PAGED_EVICTION;
        c.device = device;
        pe_engine* e = nullptr;
        const pe_status st = pe_engine_create(&c, &e);
        if (st != PE_OK) {
            sel.engines.erase(key);
            throw_status(st, "prefill_compress");
        }
        eng = e;
    }
    const std::int32_t cu[2] = {0, static_cast<std::int32_t>(L)};
    check_sync(eng, pe_prefill_prune_pack(eng, 0, K.data(), V.data(), cu, 0, 1, nullptr, nullptr),
               "prefill_compress");
    pe_info info{};
    check(pe_get_info(eng, &info), "prefill_compress");
    std::vector<std::int32_t> pages(static_cast<std::size_t>(info.max_pages));
    std::int32_t np = 0, nf = 0, ret = 0;
    check(pe_read_table(eng, 0, pages.data(), &np, &nf, &ret), "prefill_compress");
    std::vector<std::size_t> survivors;
    survivors.reserve(static_cast<std::size_t>(ret));
    std::vector<std::int32_t> pos(B);
    for (std::int32_t j = 0; j < np; ++j) {
        check(pe_read_positions(eng, pages[j], 1, pos.data(), nullptr, nullptr), "prefill_compress");
        const std::int32_t cur = j + 1 == np ? nf : static_cast<std::int32_t>(B);
        for (std::int32_t s = 0; s < cur; ++s) survivors.push_back(order[static_cast<std::size_t>(pos[s])]);
    }
    check_sync(eng, pe_table_clear(eng, 0, nullptr), "prefill_compress");
    std::sort(survivors.begin(), survivors.end());
    return survivors;
}

// PagedEvictionPolicy::evict (policy.cpp:143-155) on the device (K2).
std::int64_t EvictionPolicy::device_paged_evict(BlockTable& table, std::size_t cache_budget) {
    if (table.slot_ < 0) throw Error("BlockTable was moved from");
    auto& I = table.pool().impl();
    std::lock_guard lock(I.mu);
    if (I.eng == nullptr) return -1;
    if (cache_budget > static_cast<std::size_t>(std::numeric_limits<std::int32_t>::max()))
        throw Overflow("budget exceeds int32");
    std::int32_t victim = -1;
    table.invalidate();
    check_sync(I.eng,
               pe_table_evict(I.eng, 1, &table.slot_, static_cast<std::int32_t>(cache_budget), PE_SCORE_RECOMPUTE,
                              &victim, nullptr),
               "PagedEviction decode_step");
    return victim;
}

std::int64_t EvictionPolicy::device_token_evict(BlockTable& table, pe_token_rule rule, std::int64_t arg,
                                                std::size_t cache_budget, std::uint64_t newest_position) {
    if (table.slot_ < 0) throw Error("BlockTable was moved from");
    auto& I = table.pool().impl();
    std::lock_guard lock(I.mu);
    if (I.eng == nullptr) return -1;
    if (cache_budget > static_cast<std::size_t>(std::numeric_limits<std::int32_t>::max()))
        throw Overflow("budget exceeds int32");
    std::int64_t victim = -1;
    table.invalidate();
    const std::int64_t newest = newest_position > static_cast<std::uint64_t>(std::numeric_limits<std::int64_t>::max())
                                    ? -1
                                    : static_cast<std::int64_t>(newest_position);
    check_sync(I.eng,
               pe_table_evict_token(I.eng, table.slot_, rule, arg, static_cast<std::int32_t>(cache_budget), newest,
                                    &victim, nullptr),
               "decode_step");
    return victim;
}

std::vector<char> EvictionPolicy::device_prompt_select(const std::vector<KvVector>& tokens, pe_token_rule rule,
                                                       std::size_t k) {
    std::uint32_t W = 0;
    for (const auto& kv : tokens) W = std::max<std::uint32_t>(W, static_cast<std::uint32_t>(kv.key.size()));
    const std::size_t n = tokens.size();
    std::vector<float> K(n * W, 0.0f);
    std::vector<std::int64_t> pos(n);
    for (std::size_t i = 0; i < n; ++i) {
        std::copy(tokens[i].key.begin(), tokens[i].key.end(), K.begin() + static_cast<std::ptrdiff_t>(i * W));
        pos[i] = checked_position(tokens[i].position);
    }
    std::vector<std::uint8_t> flags(n, 0);
    std::int32_t device = 0;
    check(pe_current_device(&device), "prefill_compress");
    check(pe_prompt_select(device, rule, K.data(), static_cast<std::int32_t>(n), static_cast<std::int32_t>(W), pos.data(),
                           static_cast<std::int32_t>(k), flags.data()),
          "prefill_compress");
    return std::vector<char>(flags.begin(), flags.end());
}

namespace {

// Splits the prompt by eviction flags: survivors in input order, evicted
// positions ascending (drop_positions / rank_tokens, policy.cpp:75-101).
PrefillResult split_by_flags(std::vector<KvVector> tokens, const std::vector<char>& evict) {
    std::vector<std::uint64_t> evicted;
    std::vector<KvVector> retained;
    for (std::size_t i = 0; i < tokens.size(); ++i) {
        if (evict[i]) evicted.push_back(tokens[i].position);
        else retained.push_back(std::move(tokens[i]));
    }
    std::sort(evicted.begin(), evicted.end());
    return PrefillResult{std::move(retained), EvictionDecision::tokens(std::move(evicted), 0)};
}

// StreamingLLM (policy.cpp:158-207): prefill keeps the sinks and the recent
// window by index; decode evicts the oldest non-sink token on the device.
class DeviceStreamingLlm final : public EvictionPolicy {
public:
    using EvictionPolicy::EvictionPolicy;

protected:
    PrefillResult compress(std::vector<KvVector> tokens) const override {
        const std::size_t sinks = std::min(config_.sink_count, tokens.size());
        const std::size_t window_start = tokens.size() - (config_.cache_budget - sinks);
        std::vector<char> evict(tokens.size(), 0);
        for (std::size_t i = sinks; i < window_start; ++i) evict[i] = 1;
        return split_by_flags(std::move(tokens), evict);
    }
    EvictionDecision evict(BlockTable& table, std::uint64_t newest, std::int64_t step) override {
        const std::int64_t v = device_token_evict(table, PE_TOKEN_STREAMING,
                                                  static_cast<std::int64_t>(config_.sink_count),
                                                  config_.cache_budget, newest);
        if (v < 0) return EvictionDecision::none(step);
        return EvictionDecision::tokens({static_cast<std::uint64_t>(v)}, step);
    }
};

// InvKeyL2 / KeyDiff (policy.cpp:209-284): score-based prefill and a
// per-step token eviction, both scored on the device.
class DeviceScoredTokenPolicy final : public EvictionPolicy {
public:
    DeviceScoredTokenPolicy(PolicyConfig c, pe_token_rule rule) : EvictionPolicy(c), rule_(rule) {}

protected:
    PrefillResult compress(std::vector<KvVector> tokens) const override {
        const auto evict = device_prompt_select(tokens, rule_, tokens.size() - config_.cache_budget);
        return split_by_flags(std::move(tokens), evict);
    }
    EvictionDecision evict(BlockTable& table, std::uint64_t newest, std::int64_t step) override {
        const std::int64_t v = device_token_evict(table, rule_, 0, config_.cache_budget, newest);
        if (v < 0) return EvictionDecision::none(step);
        return EvictionDecision::tokens({static_cast<std::uint64_t>(v)}, step);
    }

private:
    pe_token_rule rule_;
};

class DevicePagedEviction final : public EvictionPolicy {
public:
    using EvictionPolicy::EvictionPolicy;

protected:
    PrefillResult compress(std::vector<KvVector> tokens) const override {
        const auto keep = device_select_survivors(tokens, config_);
        std::vector<char> kept(tokens.size(), 0);
        for (const std::size_t i : keep) kept[i] = 1;
        std::vector<std::uint64_t> evicted;
        evicted.reserve(tokens.size() - keep.size());
        std::vector<KvVector> retained;
        retained.reserve(keep.size());
        for (std::size_t i = 0; i < tokens.size(); ++i) {
            if (kept[i]) retained.push_back(std::move(tokens[i]));
            else evicted.push_back(tokens[i].position);
        }
        std::sort(evicted.begin(), evicted.end());
        return PrefillResult{std::move(retained), EvictionDecision::tokens(std::move(evicted), 0)};
    }

    EvictionDecision evict(BlockTable& table, std::uint64_t, std::int64_t step) override {
        const std::int64_t victim = device_paged_evict(table, config_.cache_budget);
        if (victim < 0) return EvictionDecision::none(step);
        return EvictionDecision::page(static_cast<std::size_t>(victim), step);
    }
};

class DeviceFullCache final : public EvictionPolicy {
public:
    using EvictionPolicy::EvictionPolicy;

protected:
    PrefillResult compress(std::vector<KvVector> tokens) const override {
        return PrefillResult{std::move(tokens), EvictionDecision::none(0)};
    }
    EvictionDecision evict(BlockTable&, std::uint64_t, std::int64_t step) override {
        return EvictionDecision::none(step);
    }
};

}  // namespace

std::unique_ptr<EvictionPolicy> make_policy(PolicyConfig config) {
    switch (config.kind) {
    case PolicyKind::PagedEviction: return std::make_unique<DevicePagedEviction>(config);
    case PolicyKind::FullCache: return std::make_unique<DeviceFullCache>(config);
    case PolicyKind::StreamingLlm: return std::make_unique<DeviceStreamingLlm>(config);
    case PolicyKind::InvKeyL2: return std::make_unique<DeviceScoredTokenPolicy>(config, PE_TOKEN_MAX_KEY_NORM);
    case PolicyKind::KeyDiff: return std::make_unique<DeviceScoredTokenPolicy>(config, PE_TOKEN_KEY_DIFF);
    }
    throw Error("unknown policy kind");
}

// ---------------------------------------------------------------- attention
AttentionDetail attend_detailed(const AttentionInputs& in) {
    if (in.table == nullptr) throw Error("attend: null table");
    const std::size_t width = static_cast<std::size_t>(in.head_count) * in.head_dim;
    if (in.query.size() != width)
        throw LengthMismatch("query length " + std::to_string(in.query.size()) +
                             " does not match head_count * head_dim = " + std::to_string(width));
    const BlockTable& t = *in.table;
    if (t.retained_len() == 0) throw EmptyCache();
    auto& I = const_cast<BlockTable&>(t).pool().impl();
    std::lock_guard lock(I.mu);
    if (width > I.width) throw LengthMismatch("cached KV width does not match head layout");
    AttentionDetail d;
    d.output.resize(width);
    d.weight_sums.resize(in.head_count);
    check_sync(I.eng,
               pe_table_attend(I.eng, t.table_id(), in.query.data(), static_cast<std::int32_t>(in.head_count),
                               static_cast<std::int32_t>(in.head_dim), d.output.data(), d.weight_sums.data(),
                               nullptr),
               "attend");
    return d;
}

std::vector<float> attend(const AttentionInputs& in) { return attend_detailed(in).output; }

double output_deviation(std::span<const float> a, std::span<const float> b) {
    if (a.size() != b.size())
        throw LengthMismatch("deviation requires equal-length vectors, got " + std::to_string(a.size()) + " and " +
                             std::to_string(b.size()));
    double diff = 0.0, ref = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        const double d = static_cast<double>(a[i]) - static_cast<double>(b[i]);
        diff += d * d;
        ref += static_cast<double>(b[i]) * static_cast<double>(b[i]);
    }
    return std::sqrt(diff) / std::max(std::sqrt(ref), 1e-12);
}

// ------------------------------------------------------------------ metrics
// metrics.cpp's emitters restated: CSV numbers in the shortest round-trip
// form (std::to_chars), JSON in the layout of the reference's JSON library
// (compact, fixed field order, doubles as shortest digits with a ".0" on
// integral values and an exponent outside 1e-5 .. 1e15, NaN as null).
namespace {

std::string csv_double(double v) {
    std::array<char, 64> buf;
    const auto res = std::to_chars(buf.data(), buf.data() + buf.size(), v);
    return std::string(buf.data(), res.ptr);
}

std::string csv_field(const std::string& f) {
    if (f.find_first_of(",\"\n") == std::string::npos) return f;
    std::string q = "\"";
    for (const char c : f) {
        if (c == '"') q += '"';
        q += c;
    }
    return q + "\"";
}

std::string json_double(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    std::array<char, 64> buf;
    const auto res = std::to_chars(buf.data(), buf.data() + buf.size(), v, std::chars_format::scientific);
    const std::string sci(buf.data(), res.ptr);  // [-]d[.ddd]e(+|-)XX
    std::string out = sci[0] == '-' ? "-" : "";
    const std::size_t m0 = out.size();
    const std::size_t epos = sci.find('e');
    std::string digits;
    for (std::size_t i = m0; i < epos; ++i)
        if (sci[i] != '.') digits += sci[i];
    const int k = static_cast<int>(digits.size());
    const int n = std::stoi(sci.substr(epos + 1)) + 1;  // decimal point after n digits
    if (k <= n && n <= 15) {
        out += digits + std::string(static_cast<std::size_t>(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out += digits.substr(0, static_cast<std::size_t>(n)) + "." + digits.substr(static_cast<std::size_t>(n));
    } else if (-4 < n && n <= 0) {
        out += "0." + std::string(static_cast<std::size_t>(-n), '0') + digits;
    } else {
        out += digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int e = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
        out += eb;
    }
    return out;
}

std::string fixed4(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.4f", v);
    return b;
}

}  // namespace

std::string emit_csv(std::span<const MetricsRecord> records) {
    std::string out =
        "policy,cache_budget,page_size,prefill_len,decode_steps,batch,layer_count,seed,"
        "prefill_evicted,evictions_total,page_evictions,token_evictions,"
        "block_table_updates,mean_fragmentation,max_fragmentation,"
        "max_fragmentation_excl_newest,mean_deviation,p95_deviation,retained_bytes,"
        "prefill_wall_ns,decode_wall_ns\n";
    for (const auto& r : records) {
        const std::string ints[] = {std::to_string(r.cache_budget), std::to_string(r.page_size),
                                    std::to_string(r.prefill_len), std::to_string(r.decode_steps),
                                    std::to_string(r.batch), std::to_string(r.layer_count), std::to_string(r.seed),
                                    std::to_string(r.prefill_evicted), std::to_string(r.evictions_total),
                                    std::to_string(r.page_evictions), std::to_string(r.token_evictions),
                                    std::to_string(r.block_table_updates)};
        out += csv_field(r.policy);
        for (const auto& x : ints) out += "," + x;
        for (const double d : {r.mean_fragmentation, r.max_fragmentation, r.max_fragmentation_excl_newest,
                               r.mean_deviation, r.p95_deviation})
            out += "," + csv_double(d);
        out += "," + std::to_string(r.retained_bytes) + "," + std::to_string(r.prefill_wall_ns) + "," +
               std::to_string(r.decode_wall_ns) + "\n";
    }
    return out;
}

std::string emit_jsonl(std::span<const StepRecord> steps) {
    std::string out;
    for (const auto& s : steps) {
        out += "{\"run\":" + std::to_string(s.run) + ",\"seq\":" + std::to_string(s.sequence) +
               ",\"layer\":" + std::to_string(s.layer) + ",\"step\":" + std::to_string(s.step) +
               ",\"retained_len\":" + std::to_string(s.retained_len) + ",\"decision\":{\"kind\":";
        switch (s.decision.kind) {
        case EvictionDecision::Kind::None: out += "null"; break;
        case EvictionDecision::Kind::Tokens: {
            out += "\"tokens\",\"positions\":[";
            for (std::size_t i = 0; i < s.decision.positions.size(); ++i)
                out += (i ? "," : "") + std::to_string(s.decision.positions[i]);
            out += "]";
            break;
        }
        case EvictionDecision::Kind::Page:
            out += "\"page\",\"logical_index\":" + std::to_string(s.decision.logical_index);
            break;
        }
        out += "},\"fragmentation\":" + json_double(s.fragmentation) + ",\"deviation\":" +
               json_double(s.deviation) + "}\n";
    }
    return out;
}

std::vector<SummaryRow> summarize(std::span<const MetricsRecord> records) {
    if (records.empty()) throw EmptyInput("summarize requires at least one record");
    std::map<std::string, SummaryRow> by_policy;
    for (const auto& r : records) {
        SummaryRow& row = by_policy[r.policy];
        row.policy = r.policy;
        row.runs += 1;
        row.evictions_total += r.evictions_total;
        row.block_table_updates += r.block_table_updates;
        row.max_fragmentation_excl_newest = std::max(row.max_fragmentation_excl_newest,
                                                     r.max_fragmentation_excl_newest);
        row.mean_deviation += r.mean_deviation;
    }
    const auto paged = by_policy.find(std::string(to_string(PolicyKind::PagedEviction)));
    const double paged_updates = paged == by_policy.end() ? 0.0 : static_cast<double>(paged->second.block_table_updates);
    std::vector<SummaryRow> rows;
    for (const PolicyKind kind : {PolicyKind::PagedEviction, PolicyKind::StreamingLlm, PolicyKind::InvKeyL2,
                                  PolicyKind::KeyDiff, PolicyKind::FullCache}) {
        const auto it = by_policy.find(std::string(to_string(kind)));
        if (it == by_policy.end()) continue;
        SummaryRow row = it->second;
        row.mean_deviation /= static_cast<double>(row.runs);
        row.cadence_ratio = paged_updates > 0.0 ? static_cast<double>(row.block_table_updates) / paged_updates
                                                : std::numeric_limits<double>::quiet_NaN();
        rows.push_back(std::move(row));
    }
    return rows;
}

std::string format_summary(std::span<const SummaryRow> rows) {
    std::string out;
    char line[256];
    std::snprintf(line, sizeof line, "%-16s%6s%11s%15s%10s%22s%16s\n", "policy", "runs", "evictions", "table_updates",
                  "cadence", "max_frag_excl_newest", "mean_deviation");
    out += line;
    for (const auto& r : rows) {
        const std::string cad = std::isnan(r.cadence_ratio) ? std::string("n/a") : fixed4(r.cadence_ratio);
        std::snprintf(line, sizeof line, "%-16s%6llu%11llu%15llu%10s%22s%16s\n", r.policy.c_str(),
                      static_cast<unsigned long long>(r.runs), static_cast<unsigned long long>(r.evictions_total),
                      static_cast<unsigned long long>(r.block_table_updates), cad.c_str(),
                      fixed4(r.max_fragmentation_excl_newest).c_str(), fixed4(r.mean_deviation).c_str());
        out += line;
    }
    return out;
}

std::vector<StepRecord> step_records(std::span<const pe_step_entry> entries, std::uint32_t page_size,
                                     std::int64_t step, std::uint32_t run) {
    std::vector<StepRecord> out;
    out.reserve(entries.size());
    for (const auto& e : entries) {
        StepRecord r;
        r.run = run;
        r.step = step;
        r.retained_len = static_cast<std::size_t>(e.retained_len);
        r.decision = e.victim >= 0 ? EvictionDecision::page(static_cast<std::size_t>(e.victim), step)
                                   : EvictionDecision::none(step);
        // block_table.cpp:48-63
        if (e.page_count > 0) {
            const double slots = static_cast<double>(e.page_count) * page_size;
            r.fragmentation = 1.0 - static_cast<double>(e.retained_len) / slots;
        }
        if (e.page_count > 1) {
            const double slots = static_cast<double>(e.page_count - 1) * page_size;
            r.fragmentation_excl_newest = 1.0 - static_cast<double>(e.retained_len - e.newest_fill) / slots;
        }
        r.deviation = std::numeric_limits<double>::quiet_NaN();
        out.push_back(std::move(r));
    }
    return out;
}

}  // namespace pagedevict

// Integration self-test for smoke checks (`__graft_entry__.smoke()` calls it
// through ctypes): one PagedEviction table through prefill_compress, 64
// decode steps and attend on the device, checked against the reference's
// invariants (policy.cpp:143-155: floor(D/B) page evictions, retained
// within (C-B, C+B], pool conservation; softmax weights sum to one).
extern "C" int pagedevict_facade_selftest(char* msg, int cap) {
    using namespace pagedevict;
    auto say = [&](const std::string& m) {
        if (msg != nullptr && cap > 0) std::snprintf(msg, static_cast<std::size_t>(cap), "%s", m.c_str());
    };
    try {
        const std::uint32_t B = 16;
        const std::size_t C = 64, w = 32, L = 200, D = 64;
        PagePool pool(C / B + 2, B);
        BlockTable table(pool);
        PolicyConfig cfg;
        cfg.cache_budget = C;
        cfg.page_size = B;
        auto policy = make_policy(cfg);
        std::uint64_t x = 0x9E3779B97F4A7C15ull;
        auto nrm = [&]() {  // deterministic pseudo-normal values
            x ^= x << 13, x ^= x >> 7, x ^= x << 17;
            return static_cast<float>(static_cast<double>(x >> 11) / 9007199254740992.0 * 2.0 - 1.0);
        };
        auto tok = [&](std::uint64_t p) {
            std::vector<float> k(w), v(w);
            for (auto& a : k) a = nrm();
            for (auto& a : v) a = nrm();
            return make_kv(std::move(k), std::move(v), p);
        };
        std::vector<KvVector> prompt;
        for (std::uint64_t i = 0; i < L; ++i) prompt.push_back(tok(i));
        auto pre = policy->prefill_compress(std::move(prompt));
        if (pre.retained.size() != C || pre.decision.positions.size() != L - C) throw Error("prefill size");
        for (auto& kv : pre.retained) table.append_token(std::move(kv));
        std::size_t evictions = 0;
        for (std::uint64_t s = 1; s <= D; ++s) {
            const auto d = policy->decode_step(table, tok(L + s - 1), static_cast<std::int64_t>(s));
            evictions += d.kind == EvictionDecision::Kind::Page;
            if (table.retained_len() > C + B || table.retained_len() <= C - B) throw Error("retained bound");
        }
        if (evictions != D / B) throw Error("expected " + std::to_string(D / B) + " page evictions");
        if (pool.allocated() + pool.free_count() != pool.capacity()) throw Error("pool conservation");
        std::vector<float> q(w);
        for (auto& a : q) a = nrm();
        const auto det = attend_detailed(AttentionInputs{q, &table, 2, static_cast<std::uint32_t>(w / 2)});
        for (const double s : det.weight_sums)
            if (std::fabs(s - 1.0) > 1e-12) throw Error("softmax weights");
        say("facade ok: " + std::to_string(evictions) + " page evictions, retained " +
            std::to_string(table.retained_len()));
        return 0;
    } catch (const std::exception& e) {
        say(e.what());
        return 1;
    }
}
