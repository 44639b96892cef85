"""o9: simulated upir.data map semantics -- TEST INFRASTRUCTURE.

Device memory is simulated as tagged byte spaces.  Mapping
kinds follow PAPER.md:792 (Fig. 5 data-mapping-property 'to' | 'from' |
'tofrom' | 'allocate'); movement direction follows PAPER.md:846 (Fig. 6
dm-direction forward | backward; reading c19: forward = host -> device).
Present-table reference counting is reading c18: the H2D copy happens on the
0 -> 1 transition (to / tofrom), the D2H copy on 1 -> 0 (from / tofrom);
'allocate' and 'from' never copy at enter and the device bytes are the
poison byte 0xA5 until written.
"""
import numpy as np

POISON = 0xA5
TO, FROM, TOFROM, ALLOC = 1, 2, 3, 4


class MapSpace:
    def __init__(self):
        self.host = {}       # name -> np.uint8 array (the host buffer)
        self.present = {}    # name -> [device bytes, refcount, kind at first enter]
        self.h2d = 0
        self.d2h = 0

    def host_buffer(self, name, data):
        self.host[name] = np.frombuffer(np.ascontiguousarray(data).tobytes(),
                                        dtype=np.uint8).copy()

    def enter(self, name, kind):
        if name in self.present:
            self.present[name][1] += 1
            return
        hb = self.host[name]
        if kind in (TO, TOFROM):
            dev = hb.copy()
            self.h2d += hb.nbytes
        else:
            dev = np.full(hb.nbytes, POISON, dtype=np.uint8)
        self.present[name] = [dev, 1, kind]

    def exit(self, name):
        if name not in self.present:
            raise KeyError("not mapped")
        ent = self.present[name]
        ent[1] -= 1
        if ent[1] == 0:
            if ent[2] in (FROM, TOFROM):
                self.host[name][:] = ent[0]
                self.d2h += ent[0].nbytes
            del self.present[name]

    def update(self, name, backward):
        dev = self.present[name][0]
        if backward:
            self.host[name][:] = dev
            self.d2h += dev.nbytes
        else:
            dev[:] = self.host[name]
            self.h2d += dev.nbytes

    def device(self, name):
        return self.present[name][0]

    def live(self):
        return len(self.present)
