// sk_tableau.h — stabilizer (tableau) shards of the native engine: the
// reference's StabilizerShard (pkg/src/shardsim/tableau.py) with bit-packed
// rows.  A shard of w <= 64 qubits is 2w rows of (x, z) 64-bit masks plus a
// phase bit (rows 0..w-1 destabilisers, w..2w-1 stabilisers); a gate is a
// handful of word operations per row and the Aaronson-Gottesman rowsum is two
// popcounts, so the tableau lives next to the engine's host bookkeeping.
// Every applied primitive is logged; converting the shard to a dense ket
// replays the log with the device kernels (sk_engine.cu `to_dense`).
#pragma once

#include <stdint.h>

#include <cmath>
#include <complex>
#include <string>
#include <vector>

namespace sktab {

using cd = std::complex<double>;

enum LogOp : uint8_t { L_H, L_S, L_X, L_Y, L_Z, L_SWAP, L_CX, L_M, L_GPHASE };

struct LogEntry {
  LogOp op;
  int a = 0, b = 0;  // qubits (b: second qubit of swap / cx target; m: outcome)
  cd phase = 1.0;
};

// Aaronson-Gottesman g summed over the qubits of bit-packed Pauli rows
// (left = (x1, z1), right = (x2, z2)); tableau.py:336-349
inline int g_count(uint64_t x1, uint64_t z1, uint64_t x2, uint64_t z2) {
  const uint64_t y1 = x1 & z1, xonly = x1 & ~z1, zonly = ~x1 & z1;
  const uint64_t plus = (y1 & z2 & ~x2) | (xonly & z2 & x2) | (zonly & x2 & ~z2);
  const uint64_t minus = (y1 & x2 & ~z2) | (xonly & z2 & ~x2) | (zonly & x2 & z2);
  return __builtin_popcountll(plus) - __builtin_popcountll(minus);
}

inline int pmod(int v, int m) { return ((v % m) + m) % m; }  // Python's %

struct Tableau {
  int w = 0;
  std::vector<uint64_t> x, z;  // [2w] row masks, bit q = qubit q
  std::vector<uint8_t> r;      // [2w]
  std::vector<LogEntry> log;

  explicit Tableau(int width = 1) : w(width), x(2 * width, 0), z(2 * width, 0), r(2 * width, 0) {
    for (int i = 0; i < w; ++i) {
      x[i] = 1ull << i;      // destabiliser X_i
      z[w + i] = 1ull << i;  // stabiliser Z_i
    }
  }

  // ---- primitive conjugation rules (tableau.py:49-88) --------------------
  void h(int q) {
    for (int i = 0; i < 2 * w; ++i) {
      const uint64_t xq = (x[i] >> q) & 1, zq = (z[i] >> q) & 1;
      r[i] ^= (uint8_t)(xq & zq);
      x[i] = (x[i] & ~(1ull << q)) | (zq << q);
      z[i] = (z[i] & ~(1ull << q)) | (xq << q);
    }
    log.push_back({L_H, q});
  }
  void s(int q) {
    for (int i = 0; i < 2 * w; ++i) {
      const uint64_t xq = (x[i] >> q) & 1, zq = (z[i] >> q) & 1;
      r[i] ^= (uint8_t)(xq & zq);
      z[i] ^= xq << q;
    }
    log.push_back({L_S, q});
  }
  void px(int q) {
    for (int i = 0; i < 2 * w; ++i) r[i] ^= (uint8_t)((z[i] >> q) & 1);
    log.push_back({L_X, q});
  }
  void py(int q) {
    for (int i = 0; i < 2 * w; ++i) r[i] ^= (uint8_t)(((x[i] ^ z[i]) >> q) & 1);
    log.push_back({L_Y, q});
  }
  void pz(int q) {
    for (int i = 0; i < 2 * w; ++i) r[i] ^= (uint8_t)((x[i] >> q) & 1);
    log.push_back({L_Z, q});
  }
  static uint64_t swapbits(uint64_t v, int a, int b) {
    const uint64_t d = ((v >> a) ^ (v >> b)) & 1;
    return v ^ (d << a) ^ (d << b);
  }
  void swap(int a, int b) {
    for (int i = 0; i < 2 * w; ++i) {
      x[i] = swapbits(x[i], a, b);
      z[i] = swapbits(z[i], a, b);
    }
    log.push_back({L_SWAP, a, b});
  }
  void cx(int c, int t) {
    for (int i = 0; i < 2 * w; ++i) {
      const uint64_t xc = (x[i] >> c) & 1, zc = (z[i] >> c) & 1, xt = (x[i] >> t) & 1, zt = (z[i] >> t) & 1;
      r[i] ^= (uint8_t)(xc & zt & (xt ^ zc ^ 1));
      x[i] ^= xc << t;
      z[i] ^= zt << c;
    }
    log.push_back({L_CX, c, t});
  }

  // controlled Pauli (0 x, 1 y, 2 z) with polarity (tableau.py:96-127)
  void ctrl_pauli(int c, int pol, int t, int which) {
    if (pol == 0) px(c);
    if (which == 0) {
      cx(c, t);
    } else if (which == 2) {
      h(t);
      cx(c, t);
      h(t);
    } else {  // CY = S(t) CX S^dag(t)
      s(t);
      s(t);
      s(t);
      cx(c, t);
      s(t);
    }
    if (pol == 0) px(c);
  }

  void apply_word(const std::string& word, int q) {  // tableau.py:133-141, leftmost first
    for (char ch : word) {
      if (ch == 'h') h(q);
      else s(q);
    }
  }
  void append_phase(cd phase) {  // tableau.py:143-146
    if (std::abs(phase - 1.0) > 1e-15) log.push_back({L_GPHASE, 0, 0, phase});
  }

  // ---- row arithmetic (tableau.py:152-189) ------------------------------------
  void rowsum(int t, int src) {
    const int g = g_count(x[src], z[src], x[t], z[t]);
    const int val = 2 * r[t] + 2 * r[src] + g;
    r[t] = (uint8_t)(pmod(val, 4) / 2);
    x[t] ^= x[src];
    z[t] ^= z[src];
  }
  int product_phase(const std::vector<int>& rows) const {  // ordered product, prefix parities
    if (rows.empty()) return 0;
    uint64_t pxm = 0, pzm = 0;
    int g = 0, rs = 0;
    for (int k : rows) {
      g += g_count(x[k], z[k], pxm, pzm);
      pxm ^= x[k];
      pzm ^= z[k];
      rs += r[k];
    }
    return pmod(2 * rs + g, 4);
  }

  // ---- measurement and queries (tableau.py:195-256) ---------------------------
  // forced < 0: a random outcome drawn by `draw` (rng.integers(0, 2));
  // returns -1 when a forced outcome contradicts a deterministic one
  template <typename Draw>
  int measure(int q, int forced, Draw draw) {
    int p = -1;
    for (int i = 0; i < w; ++i)
      if ((x[w + i] >> q) & 1) {
        p = w + i;
        break;
      }
    int outcome;
    if (p >= 0) {
      for (int i = 0; i < 2 * w; ++i)
        if (i != p && ((x[i] >> q) & 1)) rowsum(i, p);
      x[p - w] = x[p];
      z[p - w] = z[p];
      r[p - w] = r[p];
      x[p] = 0;
      z[p] = 1ull << q;
      outcome = forced < 0 ? draw() : forced;
      r[p] = (uint8_t)outcome;
    } else {
      outcome = deterministic_outcome(q);
      if (forced >= 0 && forced != outcome) return -1;
    }
    log.push_back({L_M, q, outcome});
    return outcome;
  }
  int deterministic_outcome(int q) const {
    std::vector<int> rows;
    for (int i = 0; i < w; ++i)
      if ((x[i] >> q) & 1) rows.push_back(i + w);
    return product_phase(rows) / 2;
  }
  // ('z'|'x'|'y' as 2|0|1, sign +-1) when q is a Pauli eigenstate; false if mixed
  bool deterministic_eigen(int q, int* basis, int* sign) const {
    static const int order[3] = {2, 0, 1};  // z, x, y (tableau.py:233)
    for (int b : order) {
      bool anti = false;
      for (int i = 0; i < w && !anti; ++i) {
        const uint64_t xq = (x[w + i] >> q) & 1, zq = (z[w + i] >> q) & 1;
        anti = b == 2 ? xq : b == 0 ? zq : (xq ^ zq);
      }
      if (anti) continue;
      std::vector<int> rows;
      for (int i = 0; i < w; ++i) {
        const uint64_t dx = (x[i] >> q) & 1, dz = (z[i] >> q) & 1;
        if (b == 2 ? dx : b == 0 ? dz : (dx ^ dz)) rows.push_back(i + w);
      }
      *basis = b;
      *sign = product_phase(rows) / 2 == 0 ? 1 : -1;
      return true;
    }
    return false;
  }
};

// tensor product; a keeps its positions, b shifts up by a.w (tableau.py:362-386)
inline Tableau merge(const Tableau& a, const Tableau& b) {
  const int wa = a.w, wb = b.w, w = wa + wb;
  Tableau o(w);
  for (int i = 0; i < 2 * w; ++i) o.x[i] = o.z[i] = 0, o.r[i] = 0;
  for (int i = 0; i < wa; ++i) {
    o.x[i] = a.x[i], o.z[i] = a.z[i], o.r[i] = a.r[i];
    o.x[w + i] = a.x[wa + i], o.z[w + i] = a.z[wa + i], o.r[w + i] = a.r[wa + i];
  }
  for (int i = 0; i < wb; ++i) {
    o.x[wa + i] = b.x[i] << wa, o.z[wa + i] = b.z[i] << wa, o.r[wa + i] = b.r[i];
    o.x[w + wa + i] = b.x[wb + i] << wa, o.z[w + wa + i] = b.z[wb + i] << wa, o.r[w + wa + i] = b.r[wb + i];
  }
  o.log = a.log;
  for (LogEntry e : b.log) {
    if (e.op == L_SWAP || e.op == L_CX) e.a += wa, e.b += wa;
    else if (e.op != L_GPHASE) e.a += wa;
    o.log.push_back(e);
  }
  return o;
}

// ---- single-qubit Clifford recognition (tableau.py:393-426) ----------------------
struct CliffordEntry {
  std::string word;
  cd m[4];
};

inline void mat_mul(const cd a[4], const cd b[4], cd o[4]) {
  o[0] = a[0] * b[0] + a[1] * b[2];
  o[1] = a[0] * b[1] + a[1] * b[3];
  o[2] = a[2] * b[0] + a[3] * b[2];
  o[3] = a[2] * b[1] + a[3] * b[3];
}

// canonical key: divide out the phase of the first entry with |v| > 0.4,
// round to 9 decimals (np.round(normalized, 9))
inline bool canonical_key(const cd m[4], std::vector<long long>* key) {
  int piv = -1;
  for (int i = 0; i < 4; ++i)
    if (std::abs(m[i]) > 0.4) {
      piv = i;
      break;
    }
  if (piv < 0) return false;
  const cd f = std::abs(m[piv]) / m[piv];
  key->clear();
  for (int i = 0; i < 4; ++i) {
    const cd v = m[i] * f;
    key->push_back(std::llround(v.real() * 1e9));
    key->push_back(std::llround(v.imag() * 1e9));
  }
  return true;
}

inline const std::vector<std::pair<std::vector<long long>, CliffordEntry>>& clifford_table() {
  static const std::vector<std::pair<std::vector<long long>, CliffordEntry>> table = [] {
    const double s2 = 1.0 / std::sqrt(2.0);
    const cd H[4] = {s2, s2, s2, -s2};
    const cd S[4] = {1.0, 0.0, 0.0, std::exp(cd(0, 1) * (M_PI / 2))};
    std::vector<std::pair<std::vector<long long>, CliffordEntry>> t;
    CliffordEntry id{"", {1.0, 0.0, 0.0, 1.0}};
    std::vector<long long> k;
    canonical_key(id.m, &k);
    t.push_back({k, id});
    std::vector<CliffordEntry> frontier = {id};
    while (!frontier.empty()) {
      std::vector<CliffordEntry> nxt;
      for (const auto& e : frontier)
        for (int g = 0; g < 2; ++g) {
          CliffordEntry c;
          c.word = e.word + (g == 0 ? "h" : "s");
          mat_mul(g == 0 ? H : S, e.m, c.m);
          canonical_key(c.m, &k);
          bool seen = false;
          for (auto& p : t)
            if (p.first == k) seen = true;
          if (!seen) {
            t.push_back({k, c});
            nxt.push_back(c);
          }
        }
      frontier = nxt;
    }
    return t;
  }();
  return table;
}

// (word, phase) with m == phase * word-product within 1e-12, else false
inline bool match_clifford_1q(const cd m[4], std::string* word, cd* phase) {
  // quick reject (no allocation): a Clifford 2x2 up to phase has |m_ij|^2 in {0, 1/2, 1}
  for (int i = 0; i < 4; ++i) {
    const double a = std::norm(m[i]);
    if (std::fabs(a) > 1e-9 && std::fabs(a - 0.5) > 1e-9 && std::fabs(a - 1.0) > 1e-9) return false;
  }
  std::vector<long long> k;
  if (!canonical_key(m, &k)) return false;
  for (const auto& p : clifford_table()) {
    if (p.first != k) continue;
    const cd* c = p.second.m;
    const cd tr = (std::conj(c[0]) * m[0] + std::conj(c[2]) * m[2] + std::conj(c[1]) * m[1] +
                   std::conj(c[3]) * m[3]) / 2.0;
    if (std::abs(std::abs(tr) - 1.0) > 1e-9) return false;
    const cd ph = tr / std::abs(tr);
    for (int i = 0; i < 4; ++i)
      if (std::abs(m[i] - ph * c[i]) > 1e-12) return false;
    *word = p.second.word;
    *phase = ph;
    return true;
  }
  return false;
}

}  // namespace sktab
