"""Does per-batch dedup (K2) pay on the exchange? Byte accounting on the
north star's sharded workloads (cfg4 table-wise, cfg5 row-wise), computed from
the synthetic batches themselves (a property of the input, no GPU needed).

For each N it compares, per batch:
  push    - index bytes requester -> owners: every occurrence (4 B) vs the
            unique (table,row) keys per owner (4 B) + the per-occurrence
            inverse map the owner needs to pool each bag (ceil(log2(unique
            keys of that owner)) bits, rounded up to whole bytes);
  return  - what owners send back: pooled rows (one per (bag, owner) with a
            non-empty share; f32 for table-wise, f64 partial + count for
            row-wise) vs, if dedup replaced pooling-at-the-data, one raw
            512-B row per unique key;
  hbm     - owner rows read by K4: every occurrence vs unique keys (the K4
            DRAM traffic measured by ncu sits near the unique-row bytes: the
            L2 already captures the reuse).

    python scripts/dedup_role.py [--batches 1] > profiles/r2_dedup_role.json
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from flexemb_workload import CONFIGS, DlrmBatchGen  # noqa: E402


def account(cfg_key, hb, n_gpus, mode):
    c = CONFIGS[cfg_key]
    rows = np.asarray(c["table_rows"], dtype=np.int64)
    F, B = len(hb.feature_tables), hb.batch_size
    lens = np.diff(hb.offsets)
    feat = np.repeat(np.arange(F), B)            # bag -> feature (table-major)
    occ_t = np.repeat(np.asarray(hb.feature_tables)[feat], lens)
    occ_bag = np.repeat(np.arange(F * B), lens)
    r = hb.indices.astype(np.int64)
    if mode == "tablewise":
        owner = occ_t % n_gpus
    else:  # row-wise: contiguous row ranges per GPU
        per = (rows[occ_t] + n_gpus - 1) // n_gpus
        owner = r // per
    key = occ_t * (1 << 40) + r
    nnz = r.size
    uk, first = np.unique(key, return_index=True)
    uniq = uk.size
    # (bag, owner) pairs with a non-empty share: pooled rows returned
    pairs = np.unique(occ_bag * n_gpus + owner).size
    remote = owner != 0  # requester = GPU 0 (symmetric)
    remote_u = np.unique(key[remote]).size
    pooled_b = 512 if mode == "tablewise" else 128 * 8 + 4
    pairs_remote = np.unique((occ_bag * n_gpus + owner)[remote]).size
    per_owner_u = [np.unique(key[owner == g]).size for g in range(1, n_gpus)]
    inv_b = max(1, int(np.ceil(np.log2(max(2, max(per_owner_u)))) + 7) // 8)
    return {
        "config": cfg_key, "mode": mode, "n_gpus": n_gpus, "nnz": int(nnz), "unique": int(uniq),
        "unique_frac": uniq / nnz,
        "push_bytes": {"all_occurrences": 4 * int(remote.sum()),
                       "unique_keys_plus_inverse": 4 * remote_u + inv_b * int(remote.sum()),
                       "inverse_bytes_per_occurrence": inv_b},
        "return_bytes": {"pooled_at_owner": pooled_b * pairs_remote, "raw_unique_rows": 512 * remote_u},
        "hbm_row_bytes": {"all_occurrences": 512 * nnz, "unique_rows": 512 * uniq},
        "bag_owner_pairs": int(pairs),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=1)
    a = ap.parse_args()
    out = []
    for cfg_key, mode in (("cfg4", "tablewise"), ("cfg5", "rowwise")):
        c = CONFIGS[cfg_key]
        gen = DlrmBatchGen(c["table_rows"], c["alpha"], c["batch"], (c["pooling"],) * 2 if isinstance(c["pooling"], int)
                           else c["pooling"], seed=11, permute=c.get("permute", False))
        for _ in range(a.batches):
            hb = gen.next()
            for n in (2, 4, 8):
                rec = account(cfg_key, hb, n, mode)
                p, rt = rec["push_bytes"], rec["return_bytes"]
                tot_d = p["unique_keys_plus_inverse"] + rt["pooled_at_owner"]
                tot = p["all_occurrences"] + rt["pooled_at_owner"]
                rec["nvlink_saving_if_push_deduped"] = 1 - tot_d / tot
                out.append(rec)
                print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
