"""Record GCC libgomp's static schedules as an independent pin of o2.

OpenMP's `schedule(static)` / `schedule(static, c)` is the construct UPIR's
`loop_parallel worksharing schedule(static[, chunk])` models (PAPER.md:636-646,
Fig. 3; Table 1 maps OpenMP `for` to it).  libgomp is a
third-party runtime: it shares nothing with oracle/.

Usage: python tests/golden/gen_libgomp.py [out.json]
Writes {"cases": [[T, p, c, [thread of iteration 0..T-1]], ...]}.
"""
import json
import os
import subprocess
import sys
import tempfile

PROG = r"""
#include <omp.h>
#include <stdio.h>
#include <stdlib.h>
int main(int argc, char **argv) {
  int T = atoi(argv[1]), p = atoi(argv[2]), c = atoi(argv[3]);
  int *own = (int *)malloc(sizeof(int) * (T > 0 ? T : 1));
  omp_set_dynamic(0);
  if (c <= 0) {
    #pragma omp parallel for schedule(static) num_threads(p)
    for (int i = 0; i < T; i++) own[i] = omp_get_thread_num();
  } else {
    #pragma omp parallel for schedule(static, c) num_threads(p)
    for (int i = 0; i < T; i++) own[i] = omp_get_thread_num();
  }
  for (int i = 0; i < T; i++) printf("%d ", own[i]);
  printf("\n");
  return 0;
}
"""


def compile_prog(d):
    src = os.path.join(d, "g.c")
    exe = os.path.join(d, "g")
    with open(src, "w") as f:
        f.write(PROG)
    subprocess.check_call(["gcc", "-O1", "-fopenmp", src, "-o", exe])
    return exe


def run(exe, T, p, c):
    out = subprocess.check_output([exe, str(T), str(p), str(c)],
                                  env=dict(os.environ, OMP_DYNAMIC="false"))
    return [int(v) for v in out.split()]


def cases():
    for T in range(0, 31):
        for p in range(1, 9):
            for c in (0, 1, 2, 3, 5):
                yield T, p, c
    for T, p, c in ((1000, 7, 0), (1000, 64, 0), (997, 13, 17), (4096, 3, 0), (513, 16, 4)):
        yield T, p, c


def main(path):
    with tempfile.TemporaryDirectory() as d:
        exe = compile_prog(d)
        res = [[T, p, c, run(exe, T, p, c)] for T, p, c in cases()]
    with open(path, "w") as f:
        json.dump({"_source": "GCC libgomp schedule(static[,c]) num_threads(p); "
                              "tests/golden/gen_libgomp.py", "cases": res}, f,
                  separators=(",", ":"))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else
         os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgomp_static.json"))
