"""Oracle pins against numbers the PAPER prints:
 - Table tab:datach: maximum bit widths 6 / 63 / 63 / 48 of C1..C4;
 - the simple query's memory footprints, reproduced by this
   library's canonical formats at the paper's n = 2^27 within 1 pp.
Inputs come from synth/ (DESIGN.md §4 input recipe); nothing is read from disk.
"""
import numpy as np
import pytest

import oracle as O
import synth


def test_table_datach_widths(paper_pins):
    pins = paper_pins["table_datach_max_bit_width"]
    n = 1 << 20
    cols = {"C1": synth.gen_host("C1.plain", n), "C2": synth.gen_host("C2.plain", n),
            "C3": synth.gen_host("C3.Y", n), "C4": synth.gen_host("C4.Y", n)}
    for name, v in cols.items():
        c = O.encode(v, O.STATIC_BP, 0)  # auto width = ebw(max) (D-7 / c.2)
        assert c.bit_width == pins[name], name
    # C2 under DynBP512: width 63 only in blocks holding an outlier, else 6
    v = cols["C2"]
    c = O.encode(v, O.DYN_BP, 0, 512)
    w = np.diff(c.cw.astype(np.int64))
    has_outlier = (v[: c.n_blocks * 512].reshape(-1, 512) == np.uint64((1 << 63) - 1)).any(axis=1)
    assert (w[has_outlier] == 63).all() and (w[~has_outlier] == 6).all()
    # DynBP adapts to the outliers: smaller than static BP
    assert c.footprint() < O.encode(v, O.STATIC_BP, 0).footprint()


def _footprints(xname, yname, n):
    X = synth.gen_host(xname, n)
    Y = synth.gen_host(yname, n)
    lowest = int(X.min())  # "select the (a-priori known) lowest data element"
    Xs = O.encode(X, O.STATIC_BP, 0)
    Ys = O.encode(Y, O.STATIC_BP, 0)
    Xp = O.select(Xs, O.EQ, lowest, out_fmt=O.UNCOMPR)
    Yp = O.project(Ys, Xp, 0, O.UNCOMPR)
    pos, vals = Xp.payload, Yp.payload
    fp = {"X": Xs.footprint(), "Y": Ys.footprint(), "Xp_u": Xp.footprint(), "Yp_u": Yp.footprint()}
    for tag, (f, B) in {"s": (O.STATIC_BP, 0), "d": (O.DELTA_BP, 512), "f": (O.FOR_BP, 512)}.items():
        fp["Xp_" + tag] = O.encode(pos, f, 0, B).footprint()
        fp["Yp_" + tag] = O.encode(vals, f, 0, B).footprint()
    total_u = 8 * (2 * n + pos.size + vals.size)  # purely uncompressed footprint
    return fp, total_u, pos.size / n


SCHEME = {  # (X' format, Y' format); base columns are static BP in every scheme
    "static_base_only": ("u", "u"),
    "static_all": ("s", "s"),
    "delta_intermediates": ("d", "d"),
    "for_intermediates": ("f", "f"),
}


@pytest.mark.slow
def test_simple_query_footprints(paper_pins):
    pins = paper_pins["simple_query_footprint_pct"]
    n = 1 << pins["n_log2"]
    keys = sorted({tuple(r["cols"]) for r in pins["rows"]})
    # the three cases are independent: run them in parallel worker processes
    import multiprocessing as mp
    with mp.get_context("fork").Pool(len(keys)) as pool:
        res = pool.starmap(_footprints, [(k[0], k[1], n) for k in keys])
    cache = dict(zip(keys, res))
    for row in pins["rows"]:
        fp, total_u, sel = cache[tuple(row["cols"])]
        assert abs(sel - paper_pins["select_selectivity"]["frac"]) < 0.01  # 90%
        xf, yf = SCHEME[row["scheme"]]
        pct = 100.0 * (fp["X"] + fp["Y"] + fp["Xp_" + xf] + fp["Yp_" + yf]) / total_u
        assert abs(pct - row["paper_pct"]) <= pins["tolerance_pp"], (row, pct)
    # case 3, static BP on base only: "almost no size reduction"
    fp, total_u, _ = cache[("C3.X", "C3.Y")]
    pct = 100.0 * (fp["X"] + fp["Y"] + fp["Xp_u"] + fp["Yp_u"]) / total_u
    assert pct >= pins["case3_static_base_only"]["min_pct"]
