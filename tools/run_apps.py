"""Run the application drivers (apps/drivers.py) on the GPU; one JSON line each.

usage: python tools/run_apps.py [fem] [deblur] [pps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from apps import drivers
    which = sys.argv[1:] or ["fem", "deblur", "pps"]
    for name in which:
        fn = {"fem": drivers.fem_poisson, "deblur": drivers.deblur, "pps": drivers.pps_filter}[name]
        print(json.dumps(fn()), flush=True)


if __name__ == "__main__":
    main()
