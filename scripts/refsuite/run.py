"""Run the reference's own tests (pkg/tests) against the drop-in on a GPU box.

The reference package is the sanctioned offline install under ``baseline/_ref``
(pip --target, git-ignored, travels with the gpurun snapshot); its test files are
copied next to it by ``prepare`` (in the build container, where /root/reference
exists).  Usage:
    python scripts/refsuite/run.py prepare          # build container
    python scripts/refsuite/run.py [pytest args]    # GPU box
"""

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(REF, "ref_tests")


def prepare():
    src = "/root/reference/pkg/tests"
    shutil.rmtree(TESTS, ignore_errors=True)
    shutil.copytree(src, TESTS)
    print(f"copied {src} -> {TESTS}")


def main(argv):
    if argv[:1] == ["prepare"]:
        prepare()
        return 0
    if not os.path.isdir(TESTS):
        print(f"reference tests not found under {TESTS}; run `prepare` in the build container", file=sys.stderr)
        return 5
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.dirname(os.path.abspath(__file__)), ROOT,
                                        env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", TESTS, "-p", "dropin_plugin", "-p", "no:cacheprovider",
           "--rootdir", TESTS, "-q", *argv]
    return subprocess.call(cmd, env=env, cwd=TESTS)


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
