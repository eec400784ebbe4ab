"""Golden values for the TMS cost model, produced by running the REFERENCE itself.

    python tests/golden/make_golden_tms.py      (build container only)

Imports ``ringsim.costmodel`` from /root/reference/pkg/src (read-only) and writes
``tests/golden/tms.json``: every row of the reference's packaged paper table
(``golden_rows()``) with the reference's own unrounded ``tms`` for it, plus a grid of
extra queries (all presets, several sequence lengths, sp and flop weights) and the
reference's ``tms_table`` rows.
"""

import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from ringsim import costmodel as C  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

rows = []
for r in C.golden_rows():
    q = C.TmsQuery(C.PRESETS[r.model], r.n_seq, r.mesh[1], r.flop_weight)
    rows.append({"hardware": r.hardware, "model": r.model, "mesh": list(r.mesh), "n_seq": r.n_seq,
                 "flop_weight": r.flop_weight, "table_tms": r.tms, "ref_tms": C.tms(q)})
extra = []
for name, p in C.PRESETS.items():
    for n_seq in (4096, 65536, 262144, 786432):
        for sp in (2, 4, 8):
            for w in (1.0, 2.0, 3.5):
                extra.append({"model": name, "n_seq": n_seq, "sp": sp, "flop_weight": w,
                              "ref_tms": C.tms(C.TmsQuery(p, n_seq, sp, w))})
table = [{"model": t.model, "mesh": list(t.mesh), "n_seq": t.n_seq, "tms": t.tms}
         for t in C.tms_table(list(C.PRESETS.values()), [8192, 32768, 131072], [(1, 2), (2, 4), (1, 8)],
                              2.0)]
per_token = {name: {"other": C.non_attention_flops_per_token(p),
                    "attn_32k": C.attention_flops_per_token(p, 32768)} for name, p in C.PRESETS.items()}
with open(os.path.join(HERE, "tms.json"), "w") as f:
    json.dump({"golden_rows": rows, "extra": extra, "table": table, "per_token": per_token,
               "presets": {k: [v.n_vocab, v.d_model, v.d_ff, v.n_layer, v.n_head]
                           for k, v in C.PRESETS.items()}}, f, indent=1)
print(f"wrote {len(rows)} table rows, {len(extra)} extra queries, {len(table)} tms_table rows")
