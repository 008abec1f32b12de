"""Build oracle/build/liboracle.so (test infrastructure only)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def build():
    subprocess.run(["make", "-s", "-C", HERE, "build/liboracle.so"], check=True)
    return os.path.join(HERE, "build", "liboracle.so")


if __name__ == "__main__":
    print(build())
