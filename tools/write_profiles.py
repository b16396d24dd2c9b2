"""Write committed profile summaries (profiles/*.txt) from ncu reports and launch lists in gpurun_out/.

    python tools/write_profiles.py TAG report1.ncu-rep ... [--launches launches.csv ...]
"""
import contextlib
import io
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(argv):
    tag = argv[0]
    reps, launches, mode = [], [], "rep"
    for a in argv[1:]:
        if a == "--launches":
            mode = "launch"
            continue
        (reps if mode == "rep" else launches).append(a)
    out = io.StringIO()
    with contextlib.redirect_stdout(out):
        for l in launches:
            print(f"### launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised): {os.path.basename(l)}")
            ncu_summary.launches(l)
            print()
        for r in reps:
            ncu_summary.report(r)
            print()
    path = os.path.join(ROOT, "profiles", f"ncu_{tag}.txt")
    with open(path, "w") as fh:
        fh.write(out.getvalue())
    print(path)


if __name__ == "__main__":
    main(sys.argv[1:])
