"""Regenerates tests/golden/* from the UNMODIFIED reference (oracle/_ref/ref_probe).

Run in the build container (needs /root/reference):  python tests/golden/make_goldens.py
Large trace/plan texts are split out into gzip files under tests/golden/traces/.
"""
import gzip
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
PROBE = os.path.join(ROOT, "oracle", "_ref", "ref_probe")


def main():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"])
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.check_call([PROBE, "goldens", tmp])
        for name in os.listdir(tmp):
            data = json.load(open(os.path.join(tmp, name)))
            if name == "ref_configs.json":
                for cfg, rec in data.items():
                    for key, ext in (("trace_text", "trace"), ("plan_json", "plan.json")):
                        if key in rec:
                            path = os.path.join(HERE, "traces", f"{cfg}.{ext}.gz")
                            with open(path, "wb") as raw, gzip.GzipFile(
                                    fileobj=raw, mode="wb", mtime=0, filename="") as f:
                                f.write(rec.pop(key).encode())
                            rec[key + "_file"] = os.path.relpath(path, HERE)
            with open(os.path.join(HERE, name), "w") as f:
                json.dump(data, f, indent=1, sort_keys=True)
                f.write("\n")
    print("goldens written to", HERE, file=sys.stderr)


if __name__ == "__main__":
    main()
