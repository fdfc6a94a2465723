// Batched query scan (ssb_batch.cu): a batch of up to four queries over the
// same fact table evaluated in ONE pass, with ONE shared-memory probe per
// row per dimension link for the whole batch.
//
// Per link (a fact foreign-key column joined by one or more queries of the
// batch), every probe slot carries a TUPLE of per-query codes: query q's code
// is its group-id contribution for that dimension row (codes_kernel, ssb.cu),
// or FAIL when the row fails q's dimension filters.  The distinct tuples of a
// link are few (SSB: <= 160; the filters of a query group are dials on the
// same attributes), so each link is dictionary-encoded on the device:
//
//   ids[slot]  -> uint8 / uint16 tuple id          (staged in shared memory,
//                                                    or gathered through L2)
//   dec[id]    -> uint64: 4 x 16-bit lanes, lane q  (shared memory)
//                 = query q's code, or kLaneFail
//
// The scan adds the link's decoded word into a per-row 64-bit accumulator:
// lane q then holds query q's group id (the sum of its links' contributions)
// when every link passed, and >= kLaneFail otherwise (contributions < G <=
// 4096, at most kBatchMaxLinks + kMaxFactFilters fails of 4096 each: no lane
// overflows 16 bits).  Fact filters add kLaneFail to the lanes of the queries
// they reject.  A query's row then goes to its own shared-memory u32 bins.
//
// Joint pair (BatchScan::joint01, the kernel's JP template flag): two staged
// links share one decode table indexed by id0 * n_tup1 + id1 whose entries are
// the sums of both links' entries -- one decode load per row for the pair.
//
// Compared with scan_shared_kernel (one code table per query and link, each
// probed separately) this is one probe per link instead of one per (query,
// link), and one table per link in shared memory instead of NQ: SF=100
// Q3.1-Q3.3 (200K-slot supplier link) and Q4.1-Q4.3 fit where three separate
// tables did not.
#pragma once

#include "ssb_scan.cuh"

namespace laq {
namespace scan {

constexpr int kBatchMaxQ = 4;
constexpr int kBatchMaxLinks = 6;
constexpr int kBatchMaxFilters = 4;
constexpr uint32_t kLaneFail = 4096;
constexpr unsigned long long kDictEmpty = ~0ull;

// Tuple-id table placement.
enum : int { kIdSmemU8 = 0, kIdSmemU16 = 1, kIdGlobU8 = 2, kIdGlobU16 = 3 };

struct BatchLink {
  uint32_t base, size;        // direct probe: slot = key - base, a hit iff slot < size
  int fmt;                    // kId*
  uint32_t miss;              // tuple id of "no dim row" (fails every query joining the link)
  int id_byte;                // smem byte offset of the staged id table
  int id_bytes;               // staged bytes (multiple of 16)
  const void* ids;            // the id table in global memory
  int dec_byte;               // smem byte offset of the (replicated) decode table
  int n_dec;                  // decode entries (tuple ids incl. the miss id)
  const unsigned long long* dec;
  int bm_byte;                // >= 0: smem byte offset of the any-pass bitmap (global id formats)
  int bm_bytes;
  const uint32_t* bm;
};

struct BatchScan {
  int64_t n;
  int nq;
  Col fkc[kBatchMaxLinks];
  BatchLink link[kBatchMaxLinks];
  Col ffc[kBatchMaxFilters];
  int32_t ff_lo[kBatchMaxFilters][kBatchMaxQ], ff_hi[kBatchMaxFilters][kBatchMaxQ];
  Col mc;
  int has_measure;
  int64_t G[kBatchMaxQ];
  int bins_byte[kBatchMaxQ];  // MODE 1: u32 [count G | sum G]; MODE 2: u32 [sum G]
  unsigned long long* acc[kBatchMaxQ];
  int64_t flush_every;  // grid steps between spills of the u32 bins
  int prefetch;         // L2 prefetch distance in grid steps (0: off)
  uint32_t init_lo, init_hi;  // a row's starting lanes: kLaneFail for queries that match nothing
  uint32_t fail_lo, fail_hi;  // every lane failed (rows past the end)
  uint32_t dec_shift;         // log2(8 * decode-table replication)
  int pipe;                   // the last link is L2-gathered: software-pipelined 2-row kernel
  int dec32;                  // narrow decode: 3 x 10-bit lanes in 4-byte entries (<= 3 queries, <= 3 links)
  int joint01;                // kernel links 0 and 1 (both staged) share ONE decode table at link 1, indexed
                              // id0 * n_tup1 + id1 (entry = dec0 + dec1): one decode load per row for the pair
  uint32_t n_tup1;            // link 1's tuple ids (the joint index's radix)
  uint32_t fail32;            // the narrow lanes' fail value (a power of two >= every G)
};

// ---- device dictionary build (one launch per phase for every link) ----------

struct DictLink {
  int64_t slots;
  int64_t size;                     // probe slots: ids[size] = the miss id (keys are clamped to it)
  const int32_t* code[kBatchMaxQ];  // per query: the link's code table, nullptr = query does not join it
  unsigned long long* hkeys;        // open-addressing table, kDictEmpty = free
  int32_t* hid;
  int hbits;
  void* ids;
  int idw;                          // 1 or 2 bytes per id
  uint32_t* bm;                     // any-pass bitmap (nullptr: none)
  unsigned long long* dec;
  int dec_cap;                      // entries allocated in dec
  unsigned long long miss;          // lanes of a key with no dim row
};

struct DictArgs {
  int nl, nq;
  int64_t start[kBatchMaxLinks + 1];  // flattened slot offsets, each link rounded up to 32
  DictLink l[kBatchMaxLinks];
  int* n_dec;                         // per link: tuple ids incl. the miss id
  int* overflow;
};

void launch_dict_build(laq_ctx* ctx, const DictArgs& d);
void launch_batch(laq_ctx* ctx, const BatchScan& B, int nl, int nf, int mode, size_t smem, int grid);

}  // namespace scan
}  // namespace laq
