"""Per-kernel DRAM traffic and duration of one hot-path step, from an ncu metrics CSV.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file T.csv python tools/one_step.py --steps 2 [--workers K]
    python tools/traffic.py T.csv [--key topk_k8_cr0.01] [--update profiles/traffic.json]

Sums the LAST step's launches (the capture holds --steps steps); the Top-k launch sequence
is every sg:: kernel before the merge, the merge is k_merge_ws + k_merge.
"""
import argparse
import csv
import json
from collections import OrderedDict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--key", default=None)
    ap.add_argument("--update", default=None)
    args = ap.parse_args()
    rows = [r for r in csv.reader(open(args.csv)) if len(r) > 10]
    h = rows[0]
    ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launches = OrderedDict()
    for r in rows[1:]:
        if not r[ik].startswith(("void sg::", "sg::")):
            continue
        d = launches.setdefault(r[iid], {"name": r[ik].split("(")[0].replace("void ", "")})
        d[r[im]] = float(r[iv].replace(",", ""))
    ls = list(launches.values())
    # the last step: from the last k_sample (or k_estimate) to the end
    starts = [i for i, d in enumerate(ls) if "k_sample" in d["name"]]
    step = ls[starts[-1]:] if starts else ls
    topk = [d for d in step if "merge" not in d["name"] and "stats" not in d["name"]]
    merge = [d for d in step if "merge" in d["name"]]
    def tot(ds, m):
        return sum(d.get(m, 0.0) for d in ds)
    for d in step:
        print(f"{d['name']:36s} {d.get('gpu__time_duration.sum', 0) / 1e3:9.1f} us "
              f"{(d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)) / 1e6:10.1f} MB")
    tb = tot(topk, "dram__bytes_read.sum") + tot(topk, "dram__bytes_write.sum")
    mb = tot(merge, "dram__bytes_read.sum") + tot(merge, "dram__bytes_write.sum")
    print(f"topk sequence: {tot(topk, 'gpu__time_duration.sum') / 1e3:.1f} us, {tb / 1e6:.1f} MB")
    print(f"merge:         {tot(merge, 'gpu__time_duration.sum') / 1e3:.1f} us, {mb / 1e6:.1f} MB")
    if args.update and args.key:
        data = json.loads(open(args.update).read())
        data[f"topk_{args.key}"] = int(tb)
        data[f"merge_{args.key}"] = int(mb)
        open(args.update, "w").write(json.dumps(data, indent=1) + "\n")


if __name__ == "__main__":
    main()
