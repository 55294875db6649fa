"""Rebuild profiles/traffic.json from the committed ncu summaries (profiles/*ncu*_c<k>*_<layout>.txt).

Every entry records where its figure comes from, so that bench.py can say in the bench line whether the kernel
sources changed since the capture:
  {"bytes": dram__bytes_read.sum + dram__bytes_write.sum of ONE launch, "capture": file, "commit": the commit that last wrote the capture,
   added the capture, "kernel_sha": sha1 over csrc/device/* + csrc/gen/*.cuh AT that commit (same rule as
   bench.py kernel_sources_sha()), "kernel": demangled kernel name, "ms": gpu__time_duration of the captured launch}
Usage: python tools/make_traffic.py [--head FILE ...]   (--head: these captures were taken from the working tree,
       use the sha of the sources as they are now and commit "worktree")
"""
import glob
import hashlib
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TIME = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6, "second": 1e3}


def git(*a):
    return subprocess.run(["git", "-C", ROOT, *a], capture_output=True, text=True).stdout


def sha_at(commit):
    """kernel_sources_sha() of bench.py evaluated on the tree of `commit`."""
    base = "paper_2511_15028_b200/csrc"
    names = [l.split("\t", 1)[1] for l in git("ls-tree", "-r", commit, base + "/device", base + "/gen").splitlines() if "\t" in l]
    names = [n for n in names if n.startswith(base + "/device/") or n.endswith(".cuh")]
    # bench.py sorts the concatenation device/* + gen/*.cuh by full path
    h = hashlib.sha1()
    for n in sorted(names):
        h.update(os.path.basename(n).encode())
        h.update(subprocess.run(["git", "-C", ROOT, "show", f"{commit}:{n}"], capture_output=True).stdout)
    return h.hexdigest()[:16]


def sha_worktree():
    sys.path.insert(0, ROOT)
    import bench
    return bench.kernel_sources_sha()


def parse(path):
    out = {}
    for line in open(path, errors="replace"):
        f = line.split()
        if line.startswith("Kernel Name"):
            out["kernel"] = line[len("Kernel Name"):].strip()
        elif len(f) >= 3 and f[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum") and f[1] in UNIT:
            out[f[0]] = float(f[2]) * UNIT[f[1]]
        elif len(f) >= 3 and f[0] == "gpu__time_duration.sum" and f[1] in TIME:
            out["ms"] = float(f[2]) * TIME[f[1]]
    return out


def layout_of(kernel):
    m = re.search(r"<(?:scion_gen::)?L_([A-Za-z0-9_]+)", kernel or "")
    return m.group(1).replace("_", "-") if m else None


def main():
    heads = set()
    if "--head" in sys.argv:
        heads = {os.path.basename(x) for x in sys.argv[sys.argv.index("--head") + 1:]}
    entries = {}
    order = []
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu*.txt"))):
        name = os.path.basename(p)
        m = re.search(r"_c(\d)s?_", name)
        # scaled-down captures (shared-slab) are not the bench workload; tl<K> / staged8 / coop8 are experiment variants
        if not m or "c3s" in name or re.search(r"_(tl\d+|staged8|coop8)_", name):
            continue
        d = parse(p)
        lay = layout_of(d.get("kernel"))
        if lay is None or "dram__bytes_read.sum" not in d:
            continue
        if name in heads:
            commit, when = "worktree", 1 << 62
        else:
            commit = git("log", "-1", "--format=%h", "--", "profiles/" + name).strip()
            when = int(git("log", "-1", "--format=%ct", "--", "profiles/" + name).strip() or 0)
        order.append((when, name, f"c{m.group(1)}:{lay}:1", d, commit))
    cache = {}
    for when, name, key, d, commit in sorted(order):  # the newest capture of a key wins
        if commit not in cache:
            cache[commit] = sha_worktree() if commit == "worktree" else sha_at(commit)
        entries[key] = {"bytes": int(d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0.0)), "capture": "profiles/" + name, "commit": commit,
                        "kernel_sha": cache[commit], "kernel": d.get("kernel"), "ms": d.get("ms")}
    out = {"_comment": "dram__bytes_read.sum + dram__bytes_write.sum per launch from one `ncu --set full` capture of the bench command "
                       "(tools/profile.sh); keyed workload:layout:n_gpus; rebuilt by tools/make_traffic.py"}
    out.update(dict(sorted(entries.items())))
    json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    for k, v in sorted(entries.items()):
        print(f"{k:34s} {v['bytes'] / 1e9:8.1f} GB  {v['ms'] or 0:8.2f} ms  {v['commit']:9s} {v['capture']}")


if __name__ == "__main__":
    main()
