"""Record GCC libgomp schedule(guided[, c]) iteration -> thread maps.

libgomp's guided dispatch (an independent OpenMP runtime) cuts chunks of
max(ceil(remaining/p), c) in dispatch order; consecutive chunks taken by the
same thread appear merged in an iteration -> thread map, so the starts of the
observed runs are a SUBSET of the true chunk boundaries.  Each case is run
several times (thread timing varies) to observe most boundaries.

Usage: python tests/golden/gen_libgomp_guided.py [out.json]
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
#include <unistd.h>
int main(int argc, char **argv) {
  int T = atoi(argv[1]), p = atoi(argv[2]), c = atoi(argv[3]);
  int *own = (int *)malloc(sizeof(int) * (T > 0 ? T : 1));
  omp_set_dynamic(0);
  #pragma omp parallel for schedule(guided, c) num_threads(p)
  for (int i = 0; i < T; i++) { own[i] = omp_get_thread_num(); if (i % 7 == 0) usleep(50); }
  for (int i = 0; i < T; i++) printf("%d ", own[i]);
  printf("\n");
  return 0;
}
"""


def main(path):
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "g.c"), os.path.join(d, "g")
        open(src, "w").write(PROG)
        subprocess.check_call(["gcc", "-O1", "-fopenmp", src, "-o", exe])
        cases = []
        for T, p, c in ((100, 3, 1), (257, 4, 2), (1000, 7, 5), (64, 8, 1), (500, 2, 16), (97, 5, 3)):
            starts = set()
            for _ in range(12):
                out = subprocess.check_output([exe, str(T), str(p), str(c)]).split()
                own = [int(v) for v in out]
                starts |= {i for i in range(T) if i == 0 or own[i] != own[i - 1]}
            cases.append([T, p, c, sorted(starts)])
    json.dump({"_source": "GCC libgomp schedule(guided,c) num_threads(p); observed run starts over 12 runs; "
                          "tests/golden/gen_libgomp_guided.py", "cases": cases}, open(path, "w"),
              separators=(",", ":"))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else
         os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgomp_guided.json"))
