"""Mutation check of the oracle's pins (-m "not gpu"): each entry below is a plausible
mistake in oracle/lsm_oracle.c — a flipped comparison, a dropped term, a wrong index, a
swapped operand. The test compiles the oracle with that one textual change and runs the
pin and invariant suites (tests/test_oracle_pins.py, tests/test_oracle_invariants.py)
against the mutant through ORACLE_SO_OVERRIDE: every mutant must make at least one of
them fail. A mutant that survives would mean that part of the oracle is not pinned
(DESIGN.md §4)."""
import concurrent.futures
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "lsm_oracle.c")
SAMPLER = os.path.join(ROOT, "oracle", "lsm_sampler.c")

# (name, original text, mutated text, the reading / passage the original follows)
MUTANTS = [
    ("threshold_strict", "(info - t) <= o->c.T ? ORC_NEAR", "(info - t) < o->c.T ? ORC_NEAR", "R4: Near iff d <= T"),
    ("threshold_default", "o->c.T = o->c.W / 8 > 1 ? o->c.W / 8 : 1", "o->c.T = o->c.W / 4 > 1 ? o->c.W / 4 : 1",
     "P:365 T = W/8"),
    ("no_pvp_level_swap", "case ORC_NOREUSE: return o->c.pvp ? 1 : 0;\n        case ORC_FAR:     return o->c.pvp ? 0 : 1;",
     "case ORC_NOREUSE: return 0;\n        case ORC_FAR:     return 1;", "P:434 level swap with PVP"),
    ("window_short", "return k <= t + o->c.W ? k : NONE;", "return k < t + o->c.W ? k : NONE;", "R5: window t+1..t+W"),
    ("set_index_spec", "return (v / o->c.G) % o->S;", "return v % o->S;", "R2: set = floor(v/G) mod S"),
    ("home_block", "return v % o->c.G; }", "return v * o->c.G / o->c.N; }", "R1: home = v mod G"),
    ("bypass_reversed", "ins[j] = M[nbyp + j].v;", "ins[j] = M[j].v;", "R10: bypass the smallest incoming keys"),
    ("victim_argmax", "if (w < 0 || key_less(k, best))", "if (w < 0 || key_less(best, k))",
     "P:361: evict the minimal key"),
    ("score_dropped", "k.k0 = rank_of(o, cls); k.k1 = o->score[x];", "k.k0 = rank_of(o, cls); k.k1 = 0;",
     "P:361 static score inside a level"),
    ("class_dropped", "k.k0 = rank_of(o, cls); k.k1 = o->score[x];", "k.k0 = 0; k.k1 = o->score[x];",
     "P:363-369 priority levels"),
    ("admission_unsorted", "qsort(cand, (size_t)ncand, sizeof(qent), cmp_qent_x);", "",
     "R14: admission in node order"),
    ("queue_index", "int64_t k = cand[j].reuse % o->c.W;", "int64_t k = (cand[j].reuse + 1) % o->c.W;",
     "P:410 queue = reuse mod W"),
    ("pvp_queue_t", "int64_t k = (t + 1) % o->c.W;", "int64_t k = t % o->c.W;", "R17: queue t+1 after gather(t)"),
    ("hits_unprotected", "if (tag[w] == v) { prot[w] = 1; lu[w] = t; nH++; }", "if (tag[w] == v) { lu[w] = t; nH++; }",
     "R10: hits protected for the batch"),
    ("dynamic_order", "k.k0 = 2; k.k1 = o->c.W - (info - t);", "k.k0 = 2; k.k1 = info - t;",
     "R19: reuse by descending distance"),
    ("lru_as_mru", "case ORC_LRU:    k.k1 = lu; break;", "case ORC_LRU:    k.k1 = -lu; break;", "R20: LRU key"),
    ("far_not_victim", "if (o->c.pvp && (cx == ORC_NEAR || cx == ORC_FAR))", "if (o->c.pvp && cx == ORC_NEAR)",
     "R12: lines with a next reuse go to the victim buffer"),
    ("stale_not_fresh", "if (info == FRESH || info <= t) return ORC_FRESH;", "if (info == FRESH) return ORC_FRESH;",
     "R6: a passed snapshot reuse is Fresh (P > 1)"),
    ("peer_requests_flip", "if (r != g) cnt->peer_requests++;", "if (r == g) cnt->peer_requests++;",
     "P:299 requests from other GPUs"),
    ("rr_cursor", "h->rr[s] = (w + 1) % A;", "h->rr[s] = w;", "P:612 round robin"),
    ("no_reinsert", "} else if (kd == ORC_STORAGE || o->c.reinsert) {", "} else if (kd == ORC_STORAGE) {",
     "R15: victim-buffer hits re-inserted"),
    ("bytes_by_position", "table + ids[offs[0] + i] * (int64_t)o->c.R", "table + i * (int64_t)o->c.R",
     "Part 1: out[i] = table[ids[i]]"),
    ("staging_not_cleared", "free(h->staging); h->staging = NULL; h->nstaging = 0;\n    cnt->pvp_prefetched",
     "cnt->pvp_prefetched", "P:398 prefetched rows are single-use"),
    ("pvp_unused_dropped", "if (!contains_sorted(U, nu, h->staging[j])) cnt->pvp_unused++;",
     "if (!contains_sorted(U, nu, h->staging[j])) {}", "§8(b): pvp_unused counts staged rows not requested"),
    ("pvp_unused_inverted", "if (!contains_sorted(U, nu, h->staging[j])) cnt->pvp_unused++;",
     "if (contains_sorted(U, nu, h->staging[j])) cnt->pvp_unused++;", "§8(c): pvp_unused = |staging \\ U|"),
    ("queue_not_emptied", "h->pending_prefetched = (uint64_t)h->nstaging;\n        h->qlen[k] = 0;",
     "h->pending_prefetched = (uint64_t)h->nstaging;", "§8(c): Q_g[(t+1) mod W] = ∅ after the copy"),
    ("update_period_ignored", "return o->c.P <= 1 || t % o->c.P == 0;", "return 1;", "R6: scan every P iterations"),
]


def _kill(name, old, new, tmp):
    src = open(SRC).read()
    assert src.count(old) == 1, f"{name}: pattern must occur exactly once in lsm_oracle.c"
    mdir = os.path.join(tmp, name)
    os.makedirs(mdir, exist_ok=True)
    msrc = os.path.join(mdir, "lsm_oracle.c")
    with open(msrc, "w") as f:
        f.write(src.replace(old, new))
    so = os.path.join(mdir, "liboracle.so")
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-w", "-shared", "-fPIC", "-I", os.path.join(ROOT, "oracle"),
                           "-o", so, msrc, SAMPLER])
    env = dict(os.environ, ORACLE_SO_OVERRIDE=so)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_oracle_pins.py"),
                        os.path.join(ROOT, "tests", "test_oracle_invariants.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    return r.returncode, (r.stdout + r.stderr)[-600:]


def test_every_mutant_is_killed(tmp_path):
    with concurrent.futures.ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as ex:
        futs = {m[0]: ex.submit(_kill, m[0], m[1], m[2], str(tmp_path)) for m in MUTANTS}
        res = {k: f.result() for k, f in futs.items()}
    survivors = [(k, why) for (k, _, _, why) in MUTANTS if res[k][0] == 0]
    errors = [(k, res[k]) for k in res if res[k][0] not in (0, 1)]
    assert not errors, f"mutant runs that errored instead of failing a pin: {errors}"
    assert not survivors, f"mutants no pin rejects: {survivors}"
