// TEST (host only, no GPU): b200::parse_sparse_corpus (include/skridge_b200.hpp)
// against the UNMODIFIED reference reader skridge::read_sparse_corpus
// (dataset.cpp:87-162, linked from oracle/_ref) on valid corpora and on every
// malformed-line class: same CSR arrays, labels and dimension, or the same
// exception type, line number and message.  Exit 0 iff every case agrees.
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "skridge/dataset.hpp"
#include "skridge/errors.hpp"
#include "skridge_b200.hpp"

namespace {

struct Outcome {
  std::string kind, what;
  std::size_t line = 0;
  std::vector<std::size_t> ptr, idx;
  std::vector<double> vals, labels;
  std::size_t dim = 0;
};

Outcome run_reference(const std::string& path) {
  Outcome o;
  try {
    auto ds = skridge::read_sparse_corpus(path);
    const skridge::SparseMatrix* s = ds.data.sparse();
    o.kind = "ok";
    o.dim = ds.data.rows();
    o.ptr.assign(s->col_ptr().begin(), s->col_ptr().end());
    o.idx.assign(s->row_idx().begin(), s->row_idx().end());
    o.vals = s->values();
    o.labels = ds.labels;
  } catch (const skridge::ParseError& e) {
    o.kind = "ParseError";
    o.line = e.line();
    o.what = e.what();
  } catch (const skridge::InputError& e) {
    o.kind = "InputError";
    o.what = e.what();
  } catch (const std::exception& e) {
    o.kind = "other";
    o.what = e.what();
  }
  return o;
}

Outcome run_ours(const std::string& text) {
  namespace b = skridge::b200;
  Outcome o;
  try {
    std::istringstream in(text);
    b::CsrCorpus c = b::parse_sparse_corpus(in);
    if (c.labels.empty()) throw b::InputError("corpus: no data lines");
    o.kind = "ok";
    o.dim = c.dim;
    o.ptr.assign(c.row_ptr.begin(), c.row_ptr.end());
    o.idx.assign(c.col_idx.begin(), c.col_idx.end());
    o.vals = c.vals;
    o.labels = c.labels;
  } catch (const b::ParseError& e) {
    o.kind = "ParseError";
    o.line = e.line();
    o.what = e.what();
  } catch (const b::InputError& e) {
    o.kind = "InputError";
    o.what = e.what();
  } catch (const std::exception& e) {
    o.kind = "other";
    o.what = e.what();
  }
  return o;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";
  const std::vector<std::string> cases = {
      "# a comment line\n1.5 1:0.5 3:-2 7:1e-3   # trailing comment\n-2 2:4\n\n0 1:0 4:2.5\n3.25e0 5:1 6:-0.75 9:0.125\n",
      "1 1:1\n2 3:2.5e-300 10:-7\n+3 2:+4\n",
      "\n\n# only comments\n   \n1 2:3\n",
      "1\n2\n3 1:1\n",                  // points with no features
      "x 1:1\n",                        // bad label
      "1 1:1\n2 0:3\n",                 // index 0
      "1 1:1 1:2\n",                    // repeated index
      "1 3:1 2:2\n",                    // decreasing index
      "1 1:nan\n",                      // non-finite value
      "1 1:inf\n",
      "1 a:1\n",                        // bad index
      "1 1:\n",                         // empty value
      "1 :1\n",                         // empty index
      "1 1\n",                          // missing colon
      "1 1:2x\n",                       // trailing garbage in the value
      "1 1.0:2\n",                      // non-integer index
      "1 2:1\n1 -1:1\n",                // negative index
      "1.5e 1:1\n",                     // malformed exponent in the label
      "# nothing\n",                    // no data lines
  };
  int bad = 0;
  for (std::size_t c = 0; c < cases.size(); ++c) {
    const std::string path = dir + "/corpus_case_" + std::to_string(c) + ".txt";
    {
      std::ofstream f(path);
      f << cases[c];
    }
    const Outcome r = run_reference(path), o = run_ours(cases[c]);
    bool same = r.kind == o.kind;
    if (same && r.kind == "ok")
      same = r.dim == o.dim && r.ptr == o.ptr && r.idx == o.idx && r.vals == o.vals && r.labels == o.labels;
    if (same && r.kind == "ParseError") same = r.line == o.line && r.what == o.what;
    std::printf("case %zu: reference %s%s%s | ours %s%s%s -> %s\n", c, r.kind.c_str(), r.what.empty() ? "" : ": ",
                r.what.c_str(), o.kind.c_str(), o.what.empty() ? "" : ": ", o.what.c_str(), same ? "same" : "DIFFERENT");
    bad += !same;
    std::remove(path.c_str());
  }
  std::printf("%d of %zu cases differ\n", bad, cases.size());
  return bad == 0 ? 0 : 1;
}
