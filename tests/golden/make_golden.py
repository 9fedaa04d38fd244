"""Regenerates tests/golden/scenes_bundle.json from the reference's bundled scenes.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The bundle maps scene name -> the scene's JSON object exactly as parsed from
/root/reference/proj/scenes/<name>.json (SPEC.md:567 lists the seven scenes).
Nothing at test/bench time reads /root/reference; tests compare against this
bundle, and tests/test_golden.py re-checks it against the reference when the
reference is present.
"""
import json
import os
import sys

REF = "/root/reference/proj/scenes"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scenes_bundle.json")


def main():
    if not os.path.isdir(REF):
        print("reference scenes not present; nothing to do", file=sys.stderr)
        return 1
    bundle = {}
    for fn in sorted(os.listdir(REF)):
        if fn.endswith(".json"):
            with open(os.path.join(REF, fn)) as f:
                bundle[fn[:-5]] = json.load(f)
    with open(OUT, "w") as f:
        json.dump(bundle, f, separators=(",", ":"), sort_keys=True)
    print(f"wrote {OUT}: {sorted(bundle)}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
