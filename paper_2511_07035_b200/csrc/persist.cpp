// NEXT-1: persistence and restore of a consistent checkpoint (PAPER §4.3.2, §4.4.1 P:359,
// §4.4.3).
//
//  - "the data persistence module uses multiple threads in parallel to save the model
//    parameters to disk in the background": T writer threads pwrite disjoint 64 MiB
//    blocks of the three sections, each computing the block's CRC-32 (zlib polynomial).
//  - "After the model tensors are persisted, a callback function is used to save the
//    pre-prepared checkpoint metadata ... Saving this metadata marks the completion of the
//    latest checkpoint": the data goes to `<path>.tmp`, then the CRC table and the
//    header, fsync, rename to `<path>` (atomic), then `<path>.meta.json`, then the directory's
//    `LATEST` pointer (write + fsync + rename). A crash at any point leaves either the previous
//    LATEST or the new one, never a torn checkpoint.
//  - "When loading a checkpoint, it is first read from the SSD into CPU memory and then
//    transferred to GPU memory": gck_load_checkpoint reads and verifies every block CRC;
//    the context's restore path uploads it and re-derives the bf16 working copy.
//
// File layout (little-endian; see gck_file_header in gockpt.h): [0, 4096) header; [4096, ...)
// the per-block CRC table (3 sections x nblocks uint32, padded to 4096); then master, exp_avg,
// exp_avg_sq, each 4096-byte aligned.
#include <errno.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>
#include <zlib.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

namespace gck {
namespace {

constexpr uint64_t kBlock = 64ull << 20;
constexpr uint64_t kPage = 4096;
inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

struct Layout {
    uint64_t sec_bytes, nblocks, table_off, table_bytes, sec_off[3], file_bytes;
};

Layout layout_for(uint64_t n) {
    Layout L;
    L.sec_bytes = n * 4;
    L.nblocks = (L.sec_bytes + kBlock - 1) / kBlock;
    L.table_off = kPage;
    L.table_bytes = align_up(3 * L.nblocks * 4, kPage);
    uint64_t off = L.table_off + L.table_bytes;
    for (int s = 0; s < 3; ++s) {
        L.sec_off[s] = off;
        off = align_up(off + L.sec_bytes, kPage);
    }
    L.file_bytes = off;
    return L;
}

// Version 2 (replay-on-restore): the replay log follows the version-1 layout of the same n.
struct LogLayout {
    uint64_t log_off, table_off, table_bytes, nblocks, file_bytes;
    uint64_t slice_off[GCK_K_LIMIT], slice_bytes[GCK_K_LIMIT], slice_block0[GCK_K_LIMIT];
};

LogLayout log_layout_for(const Layout &L, uint32_t K, const uint64_t *hi) {
    LogLayout G{};
    G.log_off = L.file_bytes;
    G.table_off = G.log_off + GCK_LOG_HEADER_BYTES;
    for (uint32_t i = 0; i + 1 < K; ++i) {
        G.slice_bytes[i] = hi[i] * 2;
        G.slice_block0[i] = G.nblocks;
        G.nblocks += (G.slice_bytes[i] + kBlock - 1) / kBlock;
    }
    G.table_bytes = align_up(G.nblocks * 4, kPage);
    uint64_t off = G.table_off + G.table_bytes;
    for (uint32_t i = 0; i + 1 < K; ++i) {
        G.slice_off[i] = off;
        off = align_up(off + G.slice_bytes[i], kPage);
    }
    G.file_bytes = off;
    return G;
}

static_assert(sizeof(gck_log_header) <= GCK_LOG_HEADER_BYTES, "log header page");

bool pwrite_all(int fd, const void *buf, uint64_t len, uint64_t off) {
    const char *p = static_cast<const char *>(buf);
    while (len) {
        const ssize_t w = ::pwrite(fd, p, std::min<uint64_t>(len, 1ull << 30), (off_t)off);
        if (w < 0) {
            if (errno == EINTR) continue;
            return false;
        }
        p += w;
        off += (uint64_t)w;
        len -= (uint64_t)w;
    }
    return true;
}

bool pread_all(int fd, void *buf, uint64_t len, uint64_t off) {
    char *p = static_cast<char *>(buf);
    while (len) {
        const ssize_t r = ::pread(fd, p, std::min<uint64_t>(len, 1ull << 30), (off_t)off);
        if (r < 0) {
            if (errno == EINTR) continue;
            return false;
        }
        if (r == 0) return false;  // truncated
        p += r;
        off += (uint64_t)r;
        len -= (uint64_t)r;
    }
    return true;
}

uint32_t crc32_of(const void *p, uint64_t len) {
    uLong c = crc32(0L, Z_NULL, 0);
    const Bytef *b = static_cast<const Bytef *>(p);
    while (len) {
        const uInt chunk = (uInt)std::min<uint64_t>(len, 1u << 30);
        c = crc32(c, b, chunk);
        b += chunk;
        len -= chunk;
    }
    return (uint32_t)c;
}

bool write_small_file_atomic(const std::string &path, const std::string &content) {
    const std::string tmp = path + ".tmp";
    const int fd = ::open(tmp.c_str(), O_CREAT | O_TRUNC | O_WRONLY, 0644);
    if (fd < 0) return false;
    bool ok = pwrite_all(fd, content.data(), content.size(), 0) && ::fsync(fd) == 0;
    ok = (::close(fd) == 0) && ok;
    return ok && ::rename(tmp.c_str(), path.c_str()) == 0;
}

std::string dir_of(const std::string &path) {
    const size_t k = path.find_last_of('/');
    return k == std::string::npos ? std::string(".") : path.substr(0, k);
}
std::string base_of(const std::string &path) {
    const size_t k = path.find_last_of('/');
    return k == std::string::npos ? path : path.substr(k + 1);
}

void fsync_dir(const std::string &dir) {
    const int fd = ::open(dir.c_str(), O_RDONLY | O_DIRECTORY);
    if (fd >= 0) {
        ::fsync(fd);
        ::close(fd);
    }
}

// Fault injection for the atomicity tests: GCK_FAULT_PERSIST=<k> makes the writer stop (as if
// the process died) before writing data block k, i.e. before the header/rename/metadata/LATEST.
long fault_after_blocks() {
    const char *e = getenv("GCK_FAULT_PERSIST");
    return e ? strtol(e, nullptr, 10) : -1;
}

}  // namespace

gck_status write_checkpoint_impl(const char *path, const gck_file_header *hdr_in, const float *const sec[3],
                                 int threads, const char *meta_json, gck_persist_stats *stats, std::string *err,
                                 const ReplayLog *log) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!path || !hdr_in || !sec[0] || !sec[1] || !sec[2]) {
        *err = "null argument";
        return GCK_E_INVALID;
    }
    const uint64_t n = hdr_in->n;
    const Layout L = layout_for(n);
    LogLayout G{};
    if (log) G = log_layout_for(L, log->K, log->hi);
    const uint64_t file_bytes = log ? G.file_bytes : L.file_bytes;
    const std::string final_path(path), tmp = final_path + ".tmp";
    const int fd = ::open(tmp.c_str(), O_CREAT | O_TRUNC | O_WRONLY, 0644);
    if (fd < 0) {
        *err = "open " + tmp + ": " + strerror(errno);
        return GCK_E_IO;
    }
    if (::ftruncate(fd, (off_t)file_bytes) != 0) {
        *err = std::string("ftruncate: ") + strerror(errno);
        ::close(fd);
        ::unlink(tmp.c_str());
        return GCK_E_IO;
    }
    // jobs [0, 3 nblocks): state blocks (CRC -> table); then the gradient-slice blocks (-> gtable)
    std::vector<uint32_t> table(3 * L.nblocks, 0), gtable(G.nblocks, 0);
    std::vector<uint32_t> gslice(G.nblocks);  // slice of each gradient block
    if (log)
        for (uint32_t i = 0; i + 1 < log->K; ++i)
            for (uint64_t b = G.slice_block0[i]; b < G.slice_block0[i] + (G.slice_bytes[i] + kBlock - 1) / kBlock; ++b)
                gslice[b] = i;
    const uint64_t total = 3 * L.nblocks + G.nblocks;
    std::atomic<uint64_t> next{0};
    std::atomic<bool> failed{false};
    const long fault = fault_after_blocks();
    // the blocks written last may still be cached when the next session's drains DMA-write the
    // arena (evict_budget, internal.h): their lines are evicted after the pwrite
    const uint64_t tail = evict_budget() / kBlock + 1;
    const uint64_t first_evict = total > tail ? total - tail : 0;
    auto worker = [&]() {
        bool evicted = false;
        for (;;) {
            const uint64_t j = next.fetch_add(1);
            if (j >= total || failed.load()) break;
            if (fault >= 0 && (long)j >= fault) {  // the writer "dies" before block j
                failed = true;
                break;
            }
            if (j < 3 * L.nblocks) {
                const int s = (int)(j / L.nblocks);
                const uint64_t b = j % L.nblocks;
                const uint64_t off = b * kBlock, len = std::min(kBlock, L.sec_bytes - off);
                const char *src = reinterpret_cast<const char *>(sec[s]) + off;
                table[j] = crc32_of(src, len);
                if (!pwrite_all(fd, src, len, L.sec_off[s] + off)) failed = true;
                if (j >= first_evict) {
                    evict_lines(src, len);
                    evicted = true;
                }
            } else {
                const uint64_t gb = j - 3 * L.nblocks;
                const uint32_t i = gslice[gb];
                const uint64_t off = (gb - G.slice_block0[i]) * kBlock, len = std::min(kBlock, G.slice_bytes[i] - off);
                const char *src = reinterpret_cast<const char *>(log->glog[i]) + off;
                gtable[gb] = crc32_of(src, len);
                if (!pwrite_all(fd, src, len, G.slice_off[i] + off)) failed = true;
                if (j >= first_evict) {
                    evict_lines(src, len);
                    evicted = true;
                }
            }
        }
        if (evicted) evict_fence();
    };
    if (threads <= 0) threads = std::min(16, default_threads());
    threads = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)threads, total));
    std::vector<std::thread> pool;
    for (int k = 1; k < threads; ++k) pool.emplace_back(worker);
    worker();
    for (auto &t : pool) t.join();
    if (failed) {
        ::close(fd);
        if (fault >= 0) {  // the injected fault models the writer dying: its partial .tmp stays behind
            *err = "fault injected (GCK_FAULT_PERSIST)";
            return GCK_E_ABORTED;
        }
        *err = std::string("pwrite: ") + strerror(errno);
        ::unlink(tmp.c_str());  // a failed write leaves no partial file behind
        return GCK_E_IO;
    }
    // CRC table, then the header (with its own CRC) — the last bytes of the data file
    std::vector<char> tbl(L.table_bytes, 0);
    std::memcpy(tbl.data(), table.data(), table.size() * 4);
    gck_file_header h = *hdr_in;
    std::memcpy(h.magic, GCK_FILE_MAGIC, 8);
    h.version = log ? GCK_FILE_VERSION_LOG : GCK_FILE_VERSION;
    h.header_bytes = (uint32_t)kPage;
    h.block_bytes = kBlock;
    h.nblocks = L.nblocks;
    h.table_offset = L.table_off;
    for (int s = 0; s < 3; ++s) {
        h.section_offset[s] = L.sec_off[s];
        h.section_bytes[s] = L.sec_bytes;
    }
    h.table_crc = crc32_of(tbl.data(), table.size() * 4);
    h.header_crc = 0;
    h.header_crc = crc32_of(&h, offsetof(gck_file_header, header_crc));
    std::vector<char> page(kPage, 0);
    std::memcpy(page.data(), &h, sizeof(h));
    bool ok = pwrite_all(fd, tbl.data(), tbl.size(), L.table_off);
    if (log && ok) {  // the replay log header + gradient CRC table, before the file header
        std::vector<char> gt(G.table_bytes, 0);
        if (!gtable.empty()) std::memcpy(gt.data(), gtable.data(), gtable.size() * 4);  // K = 1: no slices
        gck_log_header lh;
        std::memset(&lh, 0, sizeof(lh));
        std::memcpy(lh.magic, GCK_LOG_MAGIC, 8);
        lh.K = log->K;
        lh.t0 = log->t0;
        for (uint32_t i = 0; i < log->K; ++i) {
            lh.lo[i] = log->lo[i];
            lh.hi[i] = log->hi[i];
            lh.rec[i] = log->rec[i];
            lh.glog_offset[i] = (i + 1 < log->K) ? G.slice_off[i] : 0;
        }
        lh.glog_table_offset = G.table_off;
        lh.glog_nblocks = G.nblocks;
        lh.glog_table_crc = crc32_of(gtable.data(), gtable.size() * 4);
        lh.log_crc = crc32_of(&lh, offsetof(gck_log_header, log_crc));
        std::vector<char> lpage(GCK_LOG_HEADER_BYTES, 0);
        std::memcpy(lpage.data(), &lh, sizeof(lh));
        ok = pwrite_all(fd, gt.data(), gt.size(), G.table_off) && pwrite_all(fd, lpage.data(), lpage.size(), G.log_off);
    }
    ok = ok && pwrite_all(fd, page.data(), kPage, 0);
    const auto t_data = std::chrono::steady_clock::now();
    ok = ok && ::fsync(fd) == 0;
    ok = (::close(fd) == 0) && ok;
    if (!ok) {
        *err = std::string("write/fsync: ") + strerror(errno);
        ::unlink(tmp.c_str());
        return GCK_E_IO;
    }
    if (::rename(tmp.c_str(), final_path.c_str()) != 0) {
        *err = std::string("rename: ") + strerror(errno);
        ::unlink(tmp.c_str());
        return GCK_E_IO;
    }
    const std::string dir = dir_of(final_path);
    fsync_dir(dir);
    // metadata callback, then the LATEST pointer: the checkpoint is complete from here on
    char meta[1024];
    snprintf(meta, sizeof(meta),
             "{\"file\": \"%s\", \"version\": %u, \"step\": %llu, \"adam_t\": %llu, \"n\": %llu, \"rank\": %u, "
             "\"world\": %u, \"bytes\": %llu, \"user\": %s}\n",
             base_of(final_path).c_str(), h.version, (unsigned long long)h.step, (unsigned long long)h.adam_t,
             (unsigned long long)n, h.rank, h.world, (unsigned long long)file_bytes,
             meta_json && *meta_json ? meta_json : "null");
    if (!write_small_file_atomic(final_path + ".meta.json", meta) ||
        !write_small_file_atomic(dir + "/LATEST.rank" + std::to_string(h.rank), base_of(final_path) + "\n")) {
        *err = std::string("metadata/LATEST: ") + strerror(errno);
        return GCK_E_IO;
    }
    fsync_dir(dir);
    const auto t1 = std::chrono::steady_clock::now();
    if (stats) {
        stats->bytes = file_bytes;
        stats->threads = threads;
        stats->seconds = std::chrono::duration<double>(t1 - t0).count();
        stats->data_seconds = std::chrono::duration<double>(t_data - t0).count();
        stats->gbs = (double)(3 * L.sec_bytes) / stats->seconds / 1e9;
    }
    return GCK_OK;
}

gck_status read_header_impl(const char *path, gck_file_header *out, std::string *err) {
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) {
        *err = std::string("open: ") + strerror(errno);
        return GCK_E_IO;
    }
    std::vector<char> page(kPage);
    const bool ok = pread_all(fd, page.data(), kPage, 0);
    ::close(fd);
    if (!ok) {
        *err = "file shorter than its header";
        return GCK_E_CORRUPT;
    }
    gck_file_header h;
    std::memcpy(&h, page.data(), sizeof(h));
    if (std::memcmp(h.magic, GCK_FILE_MAGIC, 8) != 0 ||
        (h.version != GCK_FILE_VERSION && h.version != GCK_FILE_VERSION_LOG)) {
        *err = "not a GoCkpt checkpoint file (magic/version)";
        return GCK_E_CORRUPT;
    }
    if (crc32_of(&h, offsetof(gck_file_header, header_crc)) != h.header_crc) {
        *err = "header CRC mismatch";
        return GCK_E_CORRUPT;
    }
    *out = h;
    return GCK_OK;
}

std::string plan_error(uint32_t K, const uint64_t *lo, const uint64_t *hi, uint64_t n) {
    if (K < 1 || K > GCK_K_LIMIT) return "K outside 1..64";
    for (uint32_t i = 0; i < K; ++i) {
        if (lo[i] != (i ? hi[i - 1] : 0)) return "parts are not contiguous from 0";
        if (hi[i] <= lo[i]) return "empty part";
    }
    if (hi[K - 1] != n) return "parts do not cover [0, n)";
    return "";
}

namespace {

// Read + validate the replay log header of a version-2 file (fd open), and its layout.
gck_status read_log(int fd, const gck_file_header &h, gck_log_header *lh, LogLayout *G, std::string *err) {
    const Layout L = layout_for(h.n);
    std::vector<char> page(GCK_LOG_HEADER_BYTES);
    if (!pread_all(fd, page.data(), page.size(), L.file_bytes)) {
        *err = "version-2 file shorter than its replay log header";
        return GCK_E_CORRUPT;
    }
    std::memcpy(lh, page.data(), sizeof(*lh));
    if (std::memcmp(lh->magic, GCK_LOG_MAGIC, 8) != 0) {
        *err = "replay log magic mismatch";
        return GCK_E_CORRUPT;
    }
    if (crc32_of(lh, offsetof(gck_log_header, log_crc)) != lh->log_crc) {
        *err = "replay log header CRC mismatch";
        return GCK_E_CORRUPT;
    }
    const std::string pe = plan_error(lh->K, lh->lo, lh->hi, h.n);
    if (!pe.empty()) {
        *err = "replay log plan: " + pe;
        return GCK_E_CORRUPT;
    }
    if (lh->t0 + lh->K - 1 != h.step) {
        *err = "replay log t0 + K - 1 != header step";
        return GCK_E_CORRUPT;
    }
    *G = log_layout_for(L, lh->K, lh->hi);
    bool same = G->table_off == lh->glog_table_offset && G->nblocks == lh->glog_nblocks;
    for (uint32_t i = 0; i + 1 < lh->K; ++i) same = same && G->slice_off[i] == lh->glog_offset[i];
    if (!same) {
        *err = "replay log layout fields inconsistent with the plan";
        return GCK_E_CORRUPT;
    }
    return GCK_OK;
}

gck_status read_gtable(int fd, const gck_log_header &lh, std::vector<uint32_t> *gtable, std::string *err) {
    gtable->assign(lh.glog_nblocks, 0);
    if (!pread_all(fd, gtable->data(), gtable->size() * 4, lh.glog_table_offset) ||
        crc32_of(gtable->data(), gtable->size() * 4) != lh.glog_table_crc) {
        *err = "gradient CRC table unreadable or corrupt";
        return GCK_E_CORRUPT;
    }
    return GCK_OK;
}

}  // namespace

gck_status read_log_header_impl(const char *path, gck_log_header *out, std::string *err) {
    gck_file_header h;
    gck_status st = read_header_impl(path, &h, err);
    if (st != GCK_OK) return st;
    if (h.version != GCK_FILE_VERSION_LOG) {
        *err = "not a replay-on-restore (version 2) file";
        return GCK_E_INVALID;
    }
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) {
        *err = std::string("open: ") + strerror(errno);
        return GCK_E_IO;
    }
    LogLayout G;
    st = read_log(fd, h, out, &G, err);
    ::close(fd);
    return st;
}

gck_status load_checkpoint_impl(const char *path, float *const dst[3], uint64_t n, int threads,
                                gck_file_header *hdr_out, gck_persist_stats *stats, std::string *err,
                                LoadedLog *defer) {
    const auto t0 = std::chrono::steady_clock::now();
    gck_file_header h;
    gck_status st = read_header_impl(path, &h, err);
    if (st != GCK_OK) return st;
    if (h.n != n) {
        *err = "checkpoint n " + std::to_string(h.n) + " != expected " + std::to_string(n);
        return GCK_E_INVALID;
    }
    const Layout L = layout_for(n);
    if (h.nblocks != L.nblocks || h.table_offset != L.table_off) {
        *err = "layout fields inconsistent with n";
        return GCK_E_CORRUPT;
    }
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) {
        *err = std::string("open: ") + strerror(errno);
        return GCK_E_IO;
    }
    std::vector<uint32_t> table(3 * L.nblocks);
    if (!pread_all(fd, table.data(), table.size() * 4, L.table_off) ||
        crc32_of(table.data(), table.size() * 4) != h.table_crc) {
        ::close(fd);
        *err = "CRC table unreadable or corrupt";
        return GCK_E_CORRUPT;
    }
    // version 2: the replay log, its gradient slices read with the state blocks
    gck_log_header lh{};
    LogLayout G{};
    std::vector<uint32_t> gtable, gslice;
    LoadedLog local;
    LoadedLog *lg = defer ? defer : &local;
    if (h.version == GCK_FILE_VERSION_LOG) {
        if ((st = read_log(fd, h, &lh, &G, err)) != GCK_OK || (st = read_gtable(fd, lh, &gtable, err)) != GCK_OK) {
            ::close(fd);
            return st;
        }
        uint64_t need = 0, offs[GCK_K_LIMIT] = {};
        for (uint32_t i = 0; i + 1 < lh.K; ++i) {
            offs[i] = need;
            need += align_up(lh.hi[i], 128);
        }
        uint16_t *base = nullptr;
        if (lg->buf && lg->buf_elems >= need) {
            base = lg->buf;
        } else {
            lg->storage.assign(need, 0);
            base = lg->storage.data();
        }
        lg->present = true;
        lg->lh = lh;
        for (uint32_t i = 0; i + 1 < lh.K; ++i) lg->glog[i] = base + offs[i];
        gslice.assign(G.nblocks, 0);
        for (uint32_t i = 0; i + 1 < lh.K; ++i)
            for (uint64_t b = G.slice_block0[i]; b < G.slice_block0[i] + (G.slice_bytes[i] + kBlock - 1) / kBlock; ++b)
                gslice[b] = i;
    }
    const uint64_t total = 3 * L.nblocks + G.nblocks;
    std::atomic<uint64_t> next{0};
    std::atomic<int> bad{0};  // 1 = io, 2 = crc
    std::atomic<uint64_t> bad_block{0};
    auto worker = [&]() {
        for (;;) {
            const uint64_t j = next.fetch_add(1);
            if (j >= total || bad.load()) break;
            char *p;
            uint64_t len, foff;
            uint32_t want;
            if (j < 3 * L.nblocks) {
                const int s = (int)(j / L.nblocks);
                const uint64_t b = j % L.nblocks;
                const uint64_t off = b * kBlock;
                len = std::min(kBlock, L.sec_bytes - off);
                p = reinterpret_cast<char *>(dst[s]) + off;
                foff = L.sec_off[s] + off;
                want = table[j];
            } else {
                const uint64_t gb = j - 3 * L.nblocks;
                const uint32_t i = gslice[gb];
                const uint64_t off = (gb - G.slice_block0[i]) * kBlock;
                len = std::min(kBlock, G.slice_bytes[i] - off);
                p = reinterpret_cast<char *>(lg->glog[i]) + off;
                foff = G.slice_off[i] + off;
                want = gtable[gb];
            }
            if (!pread_all(fd, p, len, foff)) {
                bad = 1;
                break;
            }
            if (crc32_of(p, len) != want) {
                bad_block = j;
                bad = 2;
                break;
            }
        }
    };
    if (threads <= 0) threads = std::min(16, default_threads());
    threads = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)threads, total));
    std::vector<std::thread> pool;
    for (int k = 1; k < threads; ++k) pool.emplace_back(worker);
    worker();
    for (auto &t : pool) t.join();
    ::close(fd);
    if (bad == 1) {
        *err = "truncated or unreadable data section";
        return GCK_E_CORRUPT;
    }
    if (bad == 2) {
        *err = "data CRC mismatch in block " + std::to_string(bad_block.load());
        return GCK_E_CORRUPT;
    }
    if (h.version == GCK_FILE_VERSION_LOG && !defer) {  // replay on the host: parts j < K to S(T)
        const uint16_t *gl[GCK_K_LIMIT] = {};
        for (uint32_t i = 0; i + 1 < lh.K; ++i) gl[i] = lg->glog[i];
        st = replay_host_impl(lh.rec, lh.K, lh.lo, lh.hi, dst[0], dst[1], dst[2], gl, threads, nullptr);
        if (st != GCK_OK) {
            *err = "host replay of the loaded log failed";
            return st;
        }
    }
    if (hdr_out) *hdr_out = h;
    if (stats) {
        const auto t1 = std::chrono::steady_clock::now();
        stats->bytes = h.version == GCK_FILE_VERSION_LOG ? G.file_bytes : L.file_bytes;
        stats->threads = threads;
        stats->seconds = std::chrono::duration<double>(t1 - t0).count();
        stats->data_seconds = stats->seconds;
        stats->gbs = (double)(3 * L.sec_bytes) / stats->seconds / 1e9;
    }
    return GCK_OK;
}

// Elements [offset, offset + count) of a checkpoint file's three sections, every touched block
// read whole and CRC-verified (resharding on load: a new ZeRO-1 rank's range spans parts of old
// ranks' files; "during loading, these shards are fetched").
gck_status load_range_impl(const char *path, uint64_t offset, uint64_t count, float *const dst[3], int threads,
                           gck_file_header *hdr_out, std::string *err) {
    gck_file_header h;
    gck_status st = read_header_impl(path, &h, err);
    if (st != GCK_OK) return st;
    if (offset > h.n || count > h.n - offset) {
        *err = "range [" + std::to_string(offset) + ", +" + std::to_string(count) + ") outside n = " + std::to_string(h.n);
        return GCK_E_INVALID;
    }
    const Layout L = layout_for(h.n);
    if (h.nblocks != L.nblocks || h.table_offset != L.table_off) {
        *err = "layout fields inconsistent with n";
        return GCK_E_CORRUPT;
    }
    if (hdr_out) *hdr_out = h;
    if (count == 0) return GCK_OK;
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) {
        *err = std::string("open: ") + strerror(errno);
        return GCK_E_IO;
    }
    std::vector<uint32_t> table(3 * L.nblocks);
    if (!pread_all(fd, table.data(), table.size() * 4, L.table_off) ||
        crc32_of(table.data(), table.size() * 4) != h.table_crc) {
        ::close(fd);
        *err = "CRC table unreadable or corrupt";
        return GCK_E_CORRUPT;
    }
    const uint64_t b0 = offset * 4 / kBlock, b1 = ((offset + count) * 4 + kBlock - 1) / kBlock;
    const uint64_t nb = b1 - b0, total = 3 * nb;
    std::atomic<uint64_t> next{0};
    std::atomic<int> bad{0};
    auto worker = [&]() {
        std::vector<char> buf;
        for (;;) {
            const uint64_t j = next.fetch_add(1);
            if (j >= total || bad.load()) break;
            const int s = (int)(j / nb);
            const uint64_t b = b0 + j % nb;
            const uint64_t off = b * kBlock, len = std::min(kBlock, L.sec_bytes - off);
            buf.resize(len);
            if (!pread_all(fd, buf.data(), len, L.sec_off[s] + off)) {
                bad = 1;
                break;
            }
            if (crc32_of(buf.data(), len) != table[s * L.nblocks + b]) {
                bad = 2;
                break;
            }
            const uint64_t lo = std::max(off, offset * 4), hi = std::min(off + len, (offset + count) * 4);
            std::memcpy(reinterpret_cast<char *>(dst[s]) + (lo - offset * 4), buf.data() + (lo - off), hi - lo);
        }
    };
    if (threads <= 0) threads = std::min(16, default_threads());
    threads = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)threads, total));
    std::vector<std::thread> pool;
    for (int k = 1; k < threads; ++k) pool.emplace_back(worker);
    worker();
    for (auto &t : pool) t.join();
    if (bad) {
        ::close(fd);
        *err = bad == 1 ? "truncated or unreadable data section" : "data CRC mismatch in a touched block";
        return GCK_E_CORRUPT;
    }
    if (h.version == GCK_FILE_VERSION_LOG) {
        // the gradient slices over [offset, end), every touched block CRC-verified, then the
        // replay of the range: the update is elementwise, so a range replays on its own
        gck_log_header lh;
        LogLayout G;
        std::vector<uint32_t> gtable;
        if ((st = read_log(fd, h, &lh, &G, err)) != GCK_OK || (st = read_gtable(fd, lh, &gtable, err)) != GCK_OK) {
            ::close(fd);
            return st;
        }
        const uint64_t end = offset + count;
        std::vector<std::vector<uint16_t>> bufs(lh.K);
        const uint16_t *gl[GCK_K_LIMIT] = {};
        uint64_t rlo[GCK_K_LIMIT], rhi[GCK_K_LIMIT];
        std::vector<char> blk;
        for (uint32_t i = 0; i < lh.K; ++i) {
            rlo[i] = std::min(std::max(lh.lo[i], offset), end) - offset;
            rhi[i] = std::min(std::max(lh.hi[i], offset), end) - offset;
            if (i + 1 == lh.K) break;
            bufs[i].assign(count, 0);
            gl[i] = bufs[i].data();
            const uint64_t e1 = std::min(end, lh.hi[i]);  // slice i holds [0, hi_i)
            if (e1 <= offset) continue;
            const uint64_t bb0 = offset * 2 / kBlock, bb1 = (e1 * 2 + kBlock - 1) / kBlock;
            for (uint64_t b = bb0; b < bb1; ++b) {
                const uint64_t off = b * kBlock, len = std::min(kBlock, G.slice_bytes[i] - off);
                blk.resize(len);
                if (!pread_all(fd, blk.data(), len, G.slice_off[i] + off) ||
                    crc32_of(blk.data(), len) != gtable[G.slice_block0[i] + b]) {
                    ::close(fd);
                    *err = "gradient slice unreadable or CRC mismatch in a touched block";
                    return GCK_E_CORRUPT;
                }
                const uint64_t a = std::max(off, offset * 2), z = std::min(off + len, e1 * 2);
                std::memcpy(reinterpret_cast<char *>(bufs[i].data()) + (a - offset * 2), blk.data() + (a - off), z - a);
            }
        }
        ::close(fd);
        return replay_host_impl(lh.rec, lh.K, rlo, rhi, dst[0], dst[1], dst[2], gl, threads, nullptr);
    }
    ::close(fd);
    return GCK_OK;
}

}  // namespace gck
