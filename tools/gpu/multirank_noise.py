import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import test_gpu_multirank as T


def main():
    one_a = T._run("ipc", 1, "c2crop")[0]
    one_b = T._run("ipc", 1, "c2crop")[0]
    for sf in (True, False):
        for rep in range(2):
            many = T._run("ipc", 2, "c2crop", sync_free=sf)
            for k in range(4):
                got = np.concatenate([m["g"][k] for m in many], axis=-2)
                w = one_a["g"][k]
                print("sync_free", sf, "rep", rep, "group", k, "2proc-vs-1 %.2e" % (np.abs(got - w).max() / np.abs(w).max()),
                      "1-vs-1 %.2e" % (np.abs(one_b["g"][k] - w).max() / np.abs(w).max()),
                      "l2 %.2e" % (np.linalg.norm(got - w) / np.linalg.norm(w)))


if __name__ == "__main__":
    main()
