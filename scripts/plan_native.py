"""Run the reference planner CLI (`meshplan plan ...`) with its intra-op strategy
table (intra.py:196-238) and ILP solver (intra.py:323-401) swapped for the native
ones (paper_2201_12023_b200/ilp.py).  Plans are byte-identical to the
pure-Python planner's (tests/test_ilp_native.py); only the planning time changes:
GPT-1.3B on (1,8) at L=4 (plans/gpt13b_n8_L4) 660 s pure Python -> 7.5 s.

  python scripts/plan_native.py --reference-src /root/reference/pkg/src -- \
      plan --builder transformer:... --cluster plans/clusters/b200_1x8.json --out DIR
"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.dont_write_bytecode = True


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference-src", default="/root/reference/pkg/src")
    ap.add_argument("--python-solver", action="store_true", help="do not patch (timing baseline)")
    ap.add_argument("rest", nargs=argparse.REMAINDER)
    args = ap.parse_args()
    sys.path.insert(0, args.reference_src)
    import meshplan
    import meshplan.intra  # noqa: F401
    from meshplan import cli
    if not args.python_solver:
        from paper_2201_12023_b200 import ilp
        ilp.patch_reference(meshplan)
    rest = args.rest[1:] if args.rest[:1] == ["--"] else args.rest
    t0 = time.perf_counter()
    rc = cli.main(rest)
    print(f"planner wall time {time.perf_counter() - t0:.2f} s "
          f"({'python' if args.python_solver else 'native'} ILP solver)", file=sys.stderr)
    return rc


if __name__ == "__main__":
    sys.exit(main())
