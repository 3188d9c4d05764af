"""Mutation check of the oracle's pins (run by hand: python tests/mutate_oracle.py).

Each mutation is a plausible slip in sc_oracle.c (dropped term, wrong sign,
wrong index, flipped comparison).  The CPU pin suite must fail for every one.
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = open(os.path.join(ROOT, "oracle", "sc_oracle.c")).read()

MUTATIONS = [
    ("threshold >= instead of >", "if (z[c] > x->tau) scratch[n++] = c;", "if (z[c] >= x->tau) scratch[n++] = c;"),
    ("ascending confidence", "if (za > zb) return -1;", "if (za < zb) return -1;"),
    ("ties to larger id", "return (a < b) ? -1 : (a > b);", "return (a > b) ? -1 : (a < b);"),
    ("last list wins", "if (x->list_labels[t] == c) return j;", "if (x->list_labels[t] == c && j == x->n_lists[app]-1) return j;"),
    ("G ignores mapping", "if (cat[labels[t]] >= 0) G |= 1u << cat[labels[t]];", "G |= 1u;"),
    ("correct ignores G", "return d < n_lists && ((G >> d) & 1u);", "return d < n_lists;"),
    ("drop max(P-,theta)", "const double a = m_over ? Pm : theta;", "const double a = Pm;"),
    ("swap P+ P-", "ell = S(x->k, a - Pp);", "ell = S(x->k, Pp - a);"),
    ("y=0 term uses P+", "ell = S(x->k, Pm - theta);", "ell = S(x->k, theta - Pm);"),
    ("gradient sign", "gp = -w * d * dsigma(z[cp]); op = cp;", "gp = w * d * dsigma(z[cp]); op = cp;"),
    ("dS missing k", "return k * sigma(k * x) * sigma(-k * x);", "return sigma(k * x) * sigma(-k * x);"),
    ("P- over all W", "else                     { if (cm < 0 || z[c] > z[cm]) cm = c; }", "{ if (cm < 0 || z[c] > z[cm]) cm = c; }"),
    ("N counts G subset not intersect", "else for (int q = 0; q < 256; ++q) if (q & m) N += h[q];", "else for (int q = 0; q < 256; ++q) if ((q & m) == q) N += h[q];"),
    ("literal N non-target wrong", "N += Gi ? hit : !any_mapped;", "N += Gi ? hit : 1;"),
    ("weight inverted", "w_row[i] = (double)M / (double)N;", "w_row[i] = (double)N / (double)M;"),
    ("app-choice: last list wins", "      if (z[x->list_labels[t]] > x->tau) return j;\n  return x->n_lists[app];\n}\n\n/* k = min",
     "      if (z[x->list_labels[t]] > x->tau && j == x->n_lists[app] - 1) return j;\n  return x->n_lists[app];\n}\n\n/* k = min"),
    ("app-choice: k- includes k", "if (y && cat[c] < kk && (ckm < 0 || z[c] > z[ckm])) ckm = c;",
     "if (y && cat[c] <= kk && (ckm < 0 || z[c] > z[ckm])) ckm = c;"),
    ("app-choice: y=0 uses theta-P", "const double arg = sigma(z[cP]) - theta;", "const double arg = theta - sigma(z[cP]);"),
    ("multi-select: y term sign", "ell += S(x->k, theta - Pj);", "ell += S(x->k, Pj - theta);"),
    ("multi-select: first list only", "if (z[x->list_labels[t]] > x->tau) { m |= 1u << j; break; }",
     "if (z[x->list_labels[t]] > x->tau) { m |= 1u << j; return m; }"),
    ("sampler: weights ignored", "total += (double)count[m] * w[m];", "total += (double)count[m];"),
    ("sampler: position from u1", "int64_t pos = (int64_t)floor(u2[i] * (double)c);", "int64_t pos = (int64_t)floor(u1[i] * (double)c);"),
    ("multi-select: shared label first list only", "if (x->list_labels[t] == c) { m |= 1u << j; break; }",
     "if (x->list_labels[t] == c) { m |= 1u << j; return m; }"),
    # batch drivers (orc_eval / orc_gt_hist / orc_ranges_eval), pinned by tests/test_oracle_batch.py
    ("eval: n_incorrect counts correct rows", "if (n_incorrect) n_incorrect[a] += (uint64_t)!ok;",
     "if (n_incorrect) n_incorrect[a] += (uint64_t)ok;"),
    ("eval: hist_pred ignores the app", "if (hist_pred) hist_pred[(int64_t)a * 256 + d] += 1;",
     "if (hist_pred) hist_pred[d] += 1;"),
    ("eval: grad_scale dropped", "if (grad_val) grad_val[S_ * i + q] = gs[q] * grad_scale;",
     "if (grad_val) grad_val[S_ * i + q] = gs[q];"),
    ("eval: loss_row = ell", "if (loss_sum) loss_sum[a] += L;\n      if (loss_row) loss_row[i] = L;",
     "if (loss_sum) loss_sum[a] += L;\n      if (loss_row) loss_row[i] = ell;"),
    ("eval: loss_sum += ell", "if (loss_sum) loss_sum[a] += L;", "if (loss_sum) loss_sum[a] += ell;"),
    ("eval: gradient slots swapped", "orc_loss_row(x, ca, z, G, wi, &ell, &L, &cs[0], &gs[0], &cs[1], &gs[1]);",
     "orc_loss_row(x, ca, z, G, wi, &ell, &L, &cs[1], &gs[1], &cs[0], &gs[0]);"),
    ("eval: weight of app 0", "const double wi = w ? w[(int64_t)a * 256 + G] : 1.0;", "const double wi = w ? w[G] : 1.0;"),
    ("eval: ld ignored", "z[c] = load_z(logits, dtype, i * ld + c);", "z[c] = load_z(logits, dtype, i * C + c);"),
    ("eval: hist_gt by decision", "if (hist_gt) hist_gt[(int64_t)a * 256 + G] += 1;\n    if (loss_sum ||",
     "if (hist_gt) hist_gt[(int64_t)a * 256 + d] += 1;\n    if (loss_sum ||"),
    ("eval: bf16 widened wrong", "uint32_t u = (uint32_t)((const uint16_t*)logits)[idx] << 16;",
     "uint32_t u = (uint32_t)((const uint16_t*)logits)[idx] << 15;"),
    ("gt_hist: Multi-Select uses the compiled map", "const uint32_t G = x->order == 2 ? orc_gt_set_raw",
     "const uint32_t G = x->order == 9 ? orc_gt_set_raw"),
    ("ranges: hist_gt by decision", "if (hist_gt) hist_gt[r] += 1;", "if (hist_gt) hist_gt[d] += 1;"),
    ("ranges: n_incorrect inverted", "if (n_incorrect) n_incorrect[0] += (uint64_t)(d != r);",
     "if (n_incorrect) n_incorrect[0] += (uint64_t)(d == r);"),
    ("ranges: weight by decision", "(double)score[i], w ? w[r] : 1.0, &L, &dL);", "(double)score[i], w ? w[d] : 1.0, &L, &dL);"),
    ("ranges: grad_scale dropped", "if (grad) grad[i] = dL * grad_scale;", "if (grad) grad[i] = dL;"),
    ("ranges: loss_row holds dL", "if (loss_row) loss_row[i] = L;\n    if (grad)", "if (loss_row) loss_row[i] = dL;\n    if (grad)"),
]


def main():
    failures = []
    with tempfile.TemporaryDirectory() as td:
        for name, old, new in MUTATIONS:
            assert SRC.count(old) >= 1, name
            src = os.path.join(td, "m.c")
            so = os.path.join(td, f"m{len(failures)}_{abs(hash(name))}.so")
            open(src, "w").write(SRC.replace(old, new))
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", so, src, "-lm"])
            env = dict(os.environ, ORACLE_SO=so)
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                                "tests/test_oracle_paper.py", "tests/test_oracle_bruteforce.py",
                                "tests/test_oracle_loss.py", "tests/test_oracle_weights.py",
                                "tests/test_oracle_patterns.py", "tests/test_oracle_ranges.py",
                                "tests/test_oracle_sampler.py", "tests/test_oracle_batch.py"],
                               cwd=ROOT, env=env, capture_output=True, text=True)
            killed = r.returncode != 0
            print(f"{'KILLED ' if killed else 'SURVIVED'}  {name}")
            if not killed:
                failures.append(name)
    if failures:
        print("surviving mutations:", failures)
        sys.exit(1)


if __name__ == "__main__":
    main()
