// bin/kinetics-b200: the command-line front end (include/kin_cli.h).
#include "../../include/kin_cli.h"

int main(int argc, char** argv) { return kin_cli_main(argc, argv); }
